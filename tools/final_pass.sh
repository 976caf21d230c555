set -x
mkdir -p gpurun_out
python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/h_tests.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/h_smoke.log 2>&1
python bench.py > gpurun_out/r2h_bench.jsonl 2> gpurun_out/r2h_bench.err
python bench.py --impl reference > gpurun_out/r2h_bench_reference.jsonl 2> gpurun_out/r2h_ref.err
python tools/bench_configs.py > gpurun_out/r2h_configs.log 2>&1
python tools/bench_rows.py > gpurun_out/r2h_rows.jsonl 2> gpurun_out/r2h_rows.err
python bench.py > gpurun_out/r2h_bench2.jsonl 2>> gpurun_out/r2h_bench.err
TAG=r2h SPECS="k1:regex:k_vision_stream.*bool.1 chol:regex:k_chol_tc" bash tools/ncu_round.sh > gpurun_out/r2h_ncu.log 2>&1
cat gpurun_out/h_tests.log gpurun_out/h_smoke.log; tail -c 600 gpurun_out/r2h_bench.jsonl; tail -c 300 gpurun_out/r2h_bench2.jsonl
