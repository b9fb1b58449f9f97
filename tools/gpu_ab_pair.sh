#!/usr/bin/env bash
# INT8 GEMM layouts: CTA-pair kernel over all 256-blocks (default) vs the 1-SM 128x256-tile kernel
# (RMX_I8_NOPAIR); INT8-path parity in each, then alternating bench lines.
set -u
mkdir -p gpurun_out
for v in default nopair default nopair; do
  unset RMX_I8_NOPAIR
  [ $v = nopair ] && export RMX_I8_NOPAIR=1
  if [ ! -f gpurun_out/ab_pytest_$v.log ]; then
    timeout 900 python -m pytest tests/test_rint8.py -x -q > gpurun_out/ab_pytest_$v.log 2>&1; echo "$v pytest rc=$?"
  fi
  timeout 600 python bench.py --no-cpu-baseline --no-e2e 2>gpurun_out/ab_$v.err | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value'],2), d.get('kernel_ms'), d['clocks']['sm_mhz'], d['roofline']['frac'])"
done
