#!/usr/bin/env bash
# T-epilogue change check: parity tests touching |T|^2 / levels / photo, then the default bench line.
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/ -x -q -m gpu -k "tepi or parity or sweep or fullsize or levels or photo or collision" > gpurun_out/tc_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/tc_pytest.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],2), d.get('kernel_ms'), d['clocks']['sm_mhz'])"
