#!/usr/bin/env bash
# Persistent (dynamic block counter, RMX_I8_PERSIST - an experiment since removed from rint8.cu)
# vs the non-persistent pair GEMM: INT8 parity, DRAM bytes / L2 hit per launch (ncu) and bench lines.
set -u
mkdir -p gpurun_out
export RMX_I8_PERSIST=1
timeout 600 python -m pytest tests/test_rint8.py tests/test_gpu_edges.py -x -q > gpurun_out/pp.log 2>&1; echo "persist pytest rc=$?"; tail -2 gpurun_out/pp.log
ARGS="--steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
for v in np p; do
  if [ $v = p ]; then export RMX_I8_PERSIST=1; else unset RMX_I8_PERSIST; fi
  timeout 300 python bench.py $ARGS > gpurun_out/pl_$v.log 2>&1 && \
  timeout 600 ncu --metrics dram__bytes_read.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum --clock-control none -k regex:"oz_gemm2" -s 20 -c 2 --csv python bench.py $ARGS > gpurun_out/pn_$v.csv 2>/dev/null
  echo "$v ncu rc=$?"
  grep -E "dram__bytes_read|hit_rate|duration" gpurun_out/pn_$v.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}' | head -6
done
for v in p np p np; do
  if [ $v = p ]; then export RMX_I8_PERSIST=1; else unset RMX_I8_PERSIST; fi
  timeout 300 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value'],2), d['roofline']['frac'], d.get('kernel_ms'))"
done
