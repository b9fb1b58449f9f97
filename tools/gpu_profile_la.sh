#!/usr/bin/env bash
# One gpurun job: full ncu captures of the matching and T-epilogue kernels on the bench command
# (after the same command exited 0 without ncu), one launch each (296 darc energies).
set -u
mkdir -p gpurun_out
ARGS="--steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
TAG=${1:-r02}
python bench.py $ARGS > gpurun_out/plain_la.log 2>&1 || { echo "plain bench failed"; exit 1; }
ncu --set full --import-source on --clock-control none -k regex:tepi_kernel -s 3 -c 1 \
    -o gpurun_out/${TAG}_tepi_full python bench.py $ARGS > gpurun_out/ncu_tepi.log 2>&1
echo "ncu tepi rc=$?"
ncu --set full --import-source on --clock-control none -k regex:match_kernel -s 3 -c 1 \
    -o gpurun_out/${TAG}_match_full python bench.py $ARGS > gpurun_out/ncu_match.log 2>&1
echo "ncu match rc=$?"
