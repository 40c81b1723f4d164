#!/bin/bash
# A/B of the dense GEMM's TMA ring depth (rebuilds ts_k_dense.o per depth; GPU box).
cd "$(dirname "$0")/../paper_1912_11554_b200/csrc" || exit 1
for S in ${STAGES:-4 6 8}; do
  rm -f build/ts_k_dense.o
  make -s EXTRA=-DTS_UMMA_STAGES=$S > /dev/null 2>&1 || { echo "build failed for $S"; continue; }
  echo "== stages $S"
  (cd ../.. && DENSE_ONLY_MASS=1 TS_PROF=1 timeout 300 python tools/dense_bench.py tf32 1024 ${W:-300} ${S_:-300} 2>&1 | tail -4)
done
rm -f build/ts_k_dense.o
make -s > /dev/null 2>&1
