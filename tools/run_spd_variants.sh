#!/bin/bash
# Tensor-core SPD solve trace (n = ${N:-7665}) with each build/var_*.so swapped in (tuning sweeps).
so=paper_2512_02293_b200/_vba.so
cp $so /tmp/_vba_orig.so
for v in "$@"; do
  cp build/var_$v.so $so
  echo "== $v"
  VBA_CHOL_TRACE=1 timeout 120 python tools/spd_time.py ${N:-7665} 2 2>&1 | grep -E "POTRF|DIAG|CHAIN|span"
done
cp /tmp/_vba_orig.so $so
