#!/usr/bin/env bash
# One gpurun job: full ncu capture of the per-energy dense-LA kernels (matching, T epilogue) on the
# bench command, after the same command exited 0 without ncu (B200_PROFILING.md recipe).
set -u
mkdir -p gpurun_out
ARGS="--steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
python bench.py $ARGS > gpurun_out/plain_la.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:"match_kernel|tepi_kernel" -s 6 -c 2 \
    -o gpurun_out/prof_la python bench.py $ARGS > gpurun_out/ncu_la.log 2>&1
echo "ncu rc=$?"
tail -3 gpurun_out/ncu_la.log
