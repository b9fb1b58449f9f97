#!/usr/bin/env bash
# One gpurun job: plain bench (JSON line), then the ncu launch list and one full capture of the
# dominant kernel on the SAME command (B200_PROFILING.md recipe). Outputs under gpurun_out/.
set -u
CFG=${1:-darc}
ARGS="--config $CFG --steps 2 --warmup 3"
mkdir -p gpurun_out
python bench.py --config $CFG > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
python bench.py $ARGS > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py $ARGS > gpurun_out/ncu_launches.log 2>&1
python bench.py $ARGS > gpurun_out/plain2.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:rform_dmma -s 3 -c 1 \
    -o gpurun_out/prof_rform python bench.py $ARGS > gpurun_out/ncu_full.log 2>&1
tail -c 3000 gpurun_out/bench_default.json
