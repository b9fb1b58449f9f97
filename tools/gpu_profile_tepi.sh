#!/usr/bin/env bash
# One gpurun job: full ncu capture of the T-epilogue kernel on the bench command (after the same
# command exited 0 without ncu).
set -u
mkdir -p gpurun_out
ARGS="--steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
python bench.py $ARGS > gpurun_out/plain_t.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:tepi_kernel -s 3 -c 1 \
    -o gpurun_out/prof_tepi python bench.py $ARGS > gpurun_out/ncu_t.log 2>&1
echo "ncu rc=$?"
tail -3 gpurun_out/ncu_t.log
