#!/usr/bin/env bash
# ncu full captures of one X-residue conversion launch: tensor-core variant and dp4a variant
set -u
mkdir -p gpurun_out
TAG=${1:-conv}
ARGS="--steps 1 --warmup 3 --no-e2e --no-cpu-baseline --repeats 1"
python bench.py $ARGS > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:oz_convert -s 12 -c 1 \
    -o gpurun_out/${TAG}_tc python bench.py $ARGS > gpurun_out/${TAG}_ncu_tc.log 2>&1
echo "tc rc=$?"
RMX_I8_CONV_ALU=1 ncu --set full --import-source on --clock-control none -k regex:oz_convert -s 12 -c 1 \
    -o gpurun_out/${TAG}_alu python bench.py $ARGS > gpurun_out/${TAG}_ncu_alu.log 2>&1
echo "alu rc=$?"
