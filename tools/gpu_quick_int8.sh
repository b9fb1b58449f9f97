#!/usr/bin/env bash
# Quick INT8-path check: parity tests of the INT8 R formation, the default bench line, and the
# serialised launch list of a short bench command (kernel shares).
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_rint8.py -x -q > gpurun_out/q_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/q_pytest.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/q_bench.json 2> gpurun_out/q_bench.err; echo "bench rc=$?"
tail -1 gpurun_out/q_bench.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d.get('kernel_ms'), d['clocks'])"
ARGS="--steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/q_launches.csv \
  python bench.py $ARGS > gpurun_out/q_ncu.log 2>&1; echo "ncu rc=$?"
