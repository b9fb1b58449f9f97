#!/usr/bin/env bash
# One gpurun job: the plain bench command, then (only if it exited 0) one full ncu capture of the
# R-formation kernel on the same command (B200_PROFILING.md recipe). Outputs under gpurun_out/.
set -u
mkdir -p gpurun_out
ARGS="--steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
python bench.py $ARGS > gpurun_out/plain_rf.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:rform_dmma -s 2 -c 1 \
    -o gpurun_out/prof_rform python bench.py $ARGS > gpurun_out/ncu_rf.log 2>&1
echo "ncu rc=$?"
tail -3 gpurun_out/ncu_rf.log
