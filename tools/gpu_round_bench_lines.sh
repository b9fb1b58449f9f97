#!/usr/bin/env bash
# The round-end bench lines only (no ncu): default darc line (INT8-CRT R, e2e + oracle baseline), the
# FP64-DMMA line, the other configs and the reference arm.
set -u
mkdir -p gpurun_out
TAG=${1:-r02}
python bench.py > gpurun_out/${TAG}_bench_default.json 2> gpurun_out/${TAG}_bench_default.err
python bench.py --r-algo dmma --no-cpu-baseline > gpurun_out/${TAG}_bench_dmma.json 2> gpurun_out/${TAG}_bench_dmma.err
for c in bp fine small tiny; do
  python bench.py --config $c --no-e2e > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err
done
python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/${TAG}_bench_reference.json 2> gpurun_out/${TAG}_bench_reference.err
tail -c 300 gpurun_out/${TAG}_bench_default.json
