set -x
python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1 ; \
ncu --set full --clock-control none --import-source on -k regex:k_vision_linearize -s 4 -c 1 -o gpurun_out/prof_k1_r1 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; \
ncu --set full --clock-control none --import-source on -k regex:k_gram -s 4 -c 1 -o gpurun_out/prof_gram_r1 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_gram.log 2>&1; \
ncu --set full --clock-control none --import-source on -k regex:k_chol_update -s 200 -c 1 -o gpurun_out/prof_chol_r1 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_chol.log 2>&1; ls -la gpurun_out
