#!/usr/bin/env bash
# Power / SM-clock trace (nvidia-smi, 50 ms) across the default darc bench: R (INT8 GEMM) phases
# against the FP64 matching / T phases.
mkdir -p gpurun_out
nvidia-smi --query-gpu=timestamp,clocks.sm,power.draw,clocks_event_reasons.active --format=csv,noheader -lms 50 > gpurun_out/power_trace.csv &
SMI=$!
timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 3 --warmup 3 2> gpurun_out/power_bench.err | tail -1 | cut -c1-300; tail -3 gpurun_out/power_bench.err
kill $SMI
