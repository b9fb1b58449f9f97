#!/usr/bin/env bash
# Round profile job (one gpurun call): default bench line, then on one shorter bench command the
# ncu launch list (gpu__time_duration per launch) and one full ncu capture of each librmx kernel.
set -u
mkdir -p gpurun_out
ARGS="--steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
python bench.py $ARGS > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py $ARGS > gpurun_out/ncu_launches.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:"rform_dmma|match_kernel|tepi_kernel" \
    -s 3 -c 3 -o gpurun_out/prof_round python bench.py $ARGS > gpurun_out/ncu_full.log 2>&1
tail -c 600 gpurun_out/bench_default.json
