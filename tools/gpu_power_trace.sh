#!/usr/bin/env bash
# Power / SM-clock trace (nvidia-smi, 20 ms; instantaneous power where the driver exposes it) across
# the default darc bench: R (INT8 GEMM) phases against the FP64 matching / T phases.
mkdir -p gpurun_out
Q=timestamp,clocks.sm,power.draw.instant,clocks_event_reasons.active
nvidia-smi --query-gpu=$Q --format=csv,noheader >/dev/null 2>&1 || Q=timestamp,clocks.sm,power.draw,clocks_event_reasons.active
nvidia-smi --query-gpu=$Q --format=csv,noheader -lms 20 > gpurun_out/power_trace.csv &
SMI=$!
timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 3 --warmup 3 2> gpurun_out/power_bench.err | tail -1 | cut -c1-200
kill $SMI
echo "query: $Q"
