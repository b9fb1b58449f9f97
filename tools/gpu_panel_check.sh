#!/usr/bin/env bash
# LU panel change check: K parity subset (incl. the bounds-checked build), the phase breakdown
# (diagnostic build) and the darc bench line.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -x -q -m gpu -k "match or parity or samples or checked or virtual" > gpurun_out/pc_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pc_pytest.log
RMX_LIB=paper_1403_5524_b200/librmx_phases.so timeout 600 python tools/phases.py > gpurun_out/pc_phases.log 2>&1; echo "phases rc=$?"; head -8 gpurun_out/pc_phases.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e --repeats 1 2>gpurun_out/pc_bench.err | tail -1 > gpurun_out/pc_bench.json
python -c "import json; d=json.load(open('gpurun_out/pc_bench.json')); print(round(d['value'],2), d.get('kernel_ms'), d['clocks']['sm_mhz'])"
