#!/bin/bash
# ncu launch time of one kernel (regex $K) on config ${CFG:-1} with each build/var_*.so swapped in.
so=paper_2512_02293_b200/_vba.so
cp $so /tmp/_vba_orig.so
for v in "$@"; do
  cp build/var_$v.so $so
  ncu --metrics gpu__time_duration.sum --clock-control none --csv -k "regex:$K" --log-file /tmp/kv.csv \
    python tools/bench_configs.py --configs ${CFG:-1} --reps 1 > /dev/null 2>&1
  echo "== $v $(python tools/launch_table.py /tmp/kv.csv 2 | sed -n 2p)"
done
cp /tmp/_vba_orig.so $so
