#!/usr/bin/env bash
# INT8-CRT R formation evidence: default bench line (int8), the DMMA line, and full ncu captures of
# the INT8 GEMM and the conversion kernel on a short bench command (after it exited 0 without ncu).
set -u
mkdir -p gpurun_out
python bench.py --no-cpu-baseline > gpurun_out/bench_int8.json 2> gpurun_out/bench_int8.err
python bench.py --r-algo dmma --no-cpu-baseline --no-e2e > gpurun_out/bench_dmma.json 2> gpurun_out/bench_dmma.err
tail -c 800 gpurun_out/bench_int8.json
ARGS="--steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
python bench.py $ARGS > gpurun_out/plain_pi8.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:"oz_gemm_kernel|oz_convert_kernel" -s 40 -c 2 \
    -o gpurun_out/prof_int8 python bench.py $ARGS > gpurun_out/ncu_pi8.log 2>&1
echo "ncu rc=$?"
tail -2 gpurun_out/ncu_pi8.log
