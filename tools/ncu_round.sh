#!/bin/bash
# Round profile pass (one GPU): plain bench first, then the launch list of the same
# command, then one `ncu --set full` capture each of K1 (linearisation instance of
# k_vision_stream), the Schur Gram and the Cholesky DAG on config ${CFG:-4}.
# Usage (from the repo root, under gpurun):  TAG=r1 bash tools/ncu_round.sh
tag=${TAG:-r1}
cfg=${CFG:-4}
out=gpurun_out
mkdir -p $out
[ -n "$NOLAUNCH" ] || python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $out/ncu_plain_$tag.log 2>&1 || { echo "plain bench failed"; tail $out/ncu_plain_$tag.log; exit 1; }
[ -n "$NOLAUNCH" ] || ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_$tag.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $out/ncu_launch_$tag.log 2>&1
specs=(${SPECS:-k1:regex:k_vision_stream.*bool.1 k2:regex:k_vision_stream.*bool.0 gram:regex:k_gram< chol:regex:k_chol_tc})
for spec in "${specs[@]}"; do
  name=${spec%%:*}; filt=${spec#*:}
  ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "$filt" -s ${SKIP:-2} -c 1 \
    -o $out/prof_${name}_$tag python tools/bench_configs.py --configs $cfg --reps 1 > $out/ncu_${name}_$tag.log 2>&1
  echo "$name: $(ls -la $out/prof_${name}_$tag.ncu-rep 2>&1 | awk '{print $5}')"
done
ls -la $out
