#!/usr/bin/env bash
# Round-end measurement job (one gpurun call): the default bench line (darc, e2e + oracle baseline),
# the other configs, the reference arm, and the ncu launch list of the default command.
set -u
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
for c in bp fine small tiny; do
  python bench.py --config $c --no-e2e > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
ARGS="--steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
python bench.py $ARGS > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py $ARGS > gpurun_out/ncu_launches.log 2>&1
echo "ncu rc=$?"
tail -c 400 gpurun_out/bench_default.json
