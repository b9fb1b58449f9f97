#!/usr/bin/env bash
# Round-end evidence in one call: smoke(), the whole GPU suite, the bench lines (default darc with e2e
# and the oracle baseline, FP64-DMMA R, the other configs, the reference arm), the ncu launch list of
# the default command and full captures of the pair GEMM + tensor-core conversion (each ncu command
# after the same bench command exited 0 without ncu).
set -u
mkdir -p gpurun_out
TAG=${1:-r02g}
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
echo "smoke rc=$?"
python -m pytest tests -m gpu -q -s -rA > gpurun_out/${TAG}_pytest_gpu_full.log 2>&1
tail -1 gpurun_out/${TAG}_pytest_gpu_full.log
bash tools/gpu_round_bench_lines.sh ${TAG}
ARGS1="--steps 1 --warmup 3 --no-e2e --no-cpu-baseline --repeats 1"
python bench.py $ARGS1 > gpurun_out/${TAG}_plain1.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py $ARGS1 > gpurun_out/${TAG}_ncu_launch.log 2>&1
echo "launches rc=$?"
ncu --set full --import-source on --clock-control none -k regex:"oz_gemm2_kernel|oz_convert_tc_kernel" -s 24 -c 2 \
    -o gpurun_out/${TAG}_int8_full python bench.py $ARGS1 > gpurun_out/${TAG}_ncu_int8.log 2>&1
echo "ncu int8 rc=$?"
