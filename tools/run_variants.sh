#!/bin/bash
# Time BASELINE config(s) with each build/var_*.so swapped in for paper_2512_02293_b200/_vba.so.
# usage (repo root, under gpurun): CFGS=4 bash tools/run_variants.sh var1 var2 ...
so=paper_2512_02293_b200/_vba.so
cp $so /tmp/_vba_orig.so
for v in "$@"; do
  cp build/var_$v.so $so
  echo "== $v"
  timeout 300 python tools/bench_configs.py --configs ${CFGS:-4} --reps ${REPS:-3} 2>&1 | grep -E "solve|stages"
done
cp /tmp/_vba_orig.so $so
