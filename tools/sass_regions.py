"""Top code regions of an ncu --page source --csv --print-source sass export by warp-stall samples (profiling aid)."""
import csv,sys
rows=list(csv.reader(open(sys.argv[1])))
hdr=rows[1]; data=rows[2:]
iS=hdr.index("Warp Stall Sampling (All Samples)"); iSrc=hdr.index("Source"); iE=hdr.index("Instructions Executed")
tot=sum(float(r[iS] or 0) for r in data)
# contiguous regions of nonzero samples, merged if gap < 64 instrs
segs=[];cur=None
for i,r in enumerate(data):
    s=float(r[iS] or 0); e=float(r[iE] or 0)
    if s>0 or e>0:
        if cur and i-cur[1] < 48: cur[1]=i; cur[2]+=s; cur[3]+=e
        else:
            cur=[i,i,s,e]; segs.append(cur)
for a,b,s,e in sorted(segs,key=lambda x:-x[2])[:25]:
    print(f"{a:6d}-{b:6d} {s/tot*100:6.2f}%  exec {e:12.0f}  first: {data[a][iSrc][:50]} | last: {data[b][iSrc][:50]}")
