#!/bin/bash
# full ncu capture of the first K1 (linearisation) launch of a cfg4 solve
tag=${1:-k1}
ncu --set full --clock-control none --import-source on -k "regex:k_vision_stream" -s ${SKIP:-1} -c 1 \
  -o gpurun_out/prof_$tag python tools/bench_configs.py --configs ${CFG:-4} --reps 1 > gpurun_out/ncu_$tag.log 2>&1
tail -1 gpurun_out/ncu_$tag.log
