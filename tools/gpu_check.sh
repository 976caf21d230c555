#!/bin/bash
# standard GPU iteration: tests, Cholesky DAG trace on cfg4, config timings
python -m pytest tests -m gpu -q -x 2>&1 | tail -3
VBA_CHOL_TRACE=1 python tools/bench_configs.py --configs ${TRACE_CFG:-4} --reps 1 2>&1 | grep -A6 "chol trace" | tail -7
python tools/bench_configs.py --configs ${CFGS:-1,3,4} 2>&1 | grep -E "cfg|stages"
