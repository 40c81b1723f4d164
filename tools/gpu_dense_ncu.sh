mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_dense_op --launch-skip 1 -c 1 -o /tmp/dn -f env DENSE_ONLY_MASS=1 python tools/dense_bench.py tf32 1024 20 4 > gpurun_out/ncu_dn.log 2>&1; echo ncu=$?
ncu -i /tmp/dn.ncu-rep --page source --csv --print-source sass > /tmp/dn.csv 2>/dev/null
python tools/sass_regions.py /tmp/dn.csv > gpurun_out/dn_regions.txt 2>&1
python - <<'PY' > gpurun_out/dn_top.txt 2>&1
import csv
rows=list(csv.reader(open('/tmp/dn.csv')))
hdr=rows[1]; data=rows[2:]
iS=hdr.index("Warp Stall Sampling (All Samples)"); iSrc=hdr.index("Source")
cols=[c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
tot=sum(float(r[iS] or 0) for r in data)
top=sorted(range(len(data)),key=lambda i:-float(data[i][iS] or 0))[:60]
for i in top:
    r=data[i]; st=sorted(((float(r[hdr.index(c)] or 0),c) for c in cols),reverse=True)[:2]
    print(f"{i:6d} {float(r[iS])/tot*100:5.2f}% {r[iSrc][:70]:70s} {st}")
PY
head -30 gpurun_out/dn_regions.txt
