#!/usr/bin/env bash
# Round-end measurement job (one gpurun call): default bench line (darc, INT8-CRT R, e2e + oracle
# baseline), the FP64-DMMA line, the other configs, the reference arm, the §8(f) rows, the ncu launch
# list of the default command and full captures of the INT8 GEMM / conversion, matching and T kernels.
set -u
mkdir -p gpurun_out
TAG=${1:-r02}
python bench.py > gpurun_out/${TAG}_bench_default.json 2> gpurun_out/${TAG}_bench_default.err
python bench.py --r-algo dmma --no-cpu-baseline > gpurun_out/${TAG}_bench_dmma.json 2> gpurun_out/${TAG}_bench_dmma.err
for c in bp fine small tiny; do
  python bench.py --config $c --no-e2e > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err
done
python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/${TAG}_bench_reference.json 2> gpurun_out/${TAG}_bench_reference.err
python tools/bench_next.py > gpurun_out/${TAG}_bench_next.jsonl 2> gpurun_out/${TAG}_bench_next.err
ARGS="--steps 2 --warmup 3 --no-e2e --no-cpu-baseline --repeats 1"
python bench.py $ARGS > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py $ARGS > gpurun_out/ncu_launches.log 2>&1
echo "ncu launches rc=$?"
ARGS1="--steps 1 --warmup 3 --no-e2e --no-cpu-baseline --repeats 1"
ncu --set full --import-source on --clock-control none -k regex:"oz_gemm2|oz_convert_kernel" -s 40 -c 2 \
    -o gpurun_out/${TAG}_int8_full python bench.py $ARGS1 > gpurun_out/ncu_pi8.log 2>&1
echo "ncu int8 rc=$?"
ncu --set full --import-source on --clock-control none -k regex:tepi_kernel -s 3 -c 1 \
    -o gpurun_out/${TAG}_tepi_full python bench.py $ARGS1 > gpurun_out/ncu_tepi.log 2>&1
echo "ncu tepi rc=$?"
ncu --set full --import-source on --clock-control none -k regex:match_kernel -s 3 -c 1 \
    -o gpurun_out/${TAG}_match_full python bench.py $ARGS1 > gpurun_out/ncu_match.log 2>&1
echo "ncu match rc=$?"
tail -c 400 gpurun_out/${TAG}_bench_default.json
