#!/bin/bash
# A/B of a compile-time option of the dense kernel on the GPU box:
#   EXTRAS="-DTS_UMMA_STAGES=6 ''" bash tools/dense_ab_build.sh
cd "$(dirname "$0")/../paper_1912_11554_b200/csrc" || exit 1
eval "set -- $EXTRAS"
for X in "$@"; do
  rm -f build/ts_k_dense.o
  make -s EXTRA="$X" > /dev/null 2>&1 || { echo "build failed for '$X'"; continue; }
  echo "== EXTRA='$X'"
  (cd ../.. && DENSE_ONLY_MASS=1 TS_PROF=1 timeout 300 python tools/dense_bench.py tf32 1024 300 300 2>&1 | grep -E "dense steps|chain 0:|M/s" | tail -3)
done
rm -f build/ts_k_dense.o
make -s > /dev/null 2>&1
