#!/usr/bin/env bash
# Matching-kernel change check: parity tests touching K, the phase breakdown (diagnostic build) and
# the default bench line.
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/ -x -q -m gpu -k "match or parity or sweep or fullsize or levels or photo" > gpurun_out/mc_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/mc_pytest.log
RMX_LIB=paper_1403_5524_b200/librmx_phases.so timeout 600 python tools/phases.py > gpurun_out/mc_phases.log 2>&1; echo "phases rc=$?"; cat gpurun_out/mc_phases.log | tail -9
timeout 600 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],2), d.get('kernel_ms'), d['clocks']['sm_mhz'])"
