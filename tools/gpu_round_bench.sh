#!/usr/bin/env bash
# Round-end measurement job (one gpurun call): the default bench line (darc, INT8-CRT R, e2e + oracle
# baseline), the FP64-DMMA line, the other configs, the reference arm, the ncu launch list of the
# default command and full captures of the INT8 GEMM / conversion kernels.
set -u
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
python bench.py --r-algo dmma --no-cpu-baseline > gpurun_out/bench_dmma.json 2> gpurun_out/bench_dmma.err
for c in bp fine small tiny; do
  python bench.py --config $c --no-e2e > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
ARGS="--steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
python bench.py $ARGS > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py $ARGS > gpurun_out/ncu_launches.log 2>&1
echo "ncu launches rc=$?"
ARGS1="--steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
python bench.py $ARGS1 > gpurun_out/plain1.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:"oz_gemm|oz_convert_kernel" -s 40 -c 4 \
    -o gpurun_out/prof_int8 python bench.py $ARGS1 > gpurun_out/ncu_pi8.log 2>&1
echo "ncu full rc=$?"
tail -c 600 gpurun_out/bench_default.json
