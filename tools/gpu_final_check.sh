#!/usr/bin/env bash
# Final job of a round: smoke(), the whole GPU suite, the default bench line, and fresh ncu captures
# of the T epilogue and matching kernels (after the bench command exited 0 without ncu).
set -u
mkdir -p gpurun_out
TAG=${1:-r02}
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
python -m pytest tests -m gpu -q -s -rA > gpurun_out/${TAG}_pytest_gpu_full.log 2>&1
tail -3 gpurun_out/${TAG}_pytest_gpu_full.log
ARGS1="--steps 1 --warmup 3 --no-e2e --no-cpu-baseline --repeats 1"
python bench.py $ARGS1 > gpurun_out/plain1.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:tepi_kernel -s 3 -c 1 \
    -o gpurun_out/${TAG}_tepi_full python bench.py $ARGS1 > gpurun_out/ncu_tepi.log 2>&1
echo "ncu tepi rc=$?"
ncu --set full --import-source on --clock-control none -k regex:match_kernel -s 3 -c 1 \
    -o gpurun_out/${TAG}_match_full python bench.py $ARGS1 > gpurun_out/ncu_match.log 2>&1
echo "ncu match rc=$?"
