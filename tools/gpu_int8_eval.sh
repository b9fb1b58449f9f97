#!/usr/bin/env bash
# INT8-CRT R formation: parity tests, bench line, launch list (shares of the INT8 path's kernels).
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_rint8.py -q -x > gpurun_out/pytest_i8.log 2>&1; tail -2 gpurun_out/pytest_i8.log
python bench.py --r-algo int8 --no-cpu-baseline --no-e2e > gpurun_out/bench_i8.json 2> gpurun_out/bench_i8.err
tail -c 1500 gpurun_out/bench_i8.json
ARGS="--r-algo int8 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
python bench.py $ARGS > gpurun_out/plain_i8.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_i8.csv \
    python bench.py $ARGS > gpurun_out/ncu_i8.log 2>&1
echo "ncu rc=$?"
