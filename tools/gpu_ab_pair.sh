#!/usr/bin/env bash
# INT8 GEMM: CTA-pair kernel vs 1-SM kernel only (RMX_I8_NOPAIR), parity tests then A/B bench lines.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_rint8.py -x -q > gpurun_out/ab_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/ab_pytest.log
for v in pair nopair pair nopair; do
  if [ $v = nopair ]; then export RMX_I8_NOPAIR=1; else unset RMX_I8_NOPAIR; fi
  timeout 600 python bench.py --no-cpu-baseline --no-e2e 2>gpurun_out/ab_$v.err | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value'],2), d.get('kernel_ms'), d['clocks']['sm_mhz'], d['roofline']['frac'])"
done
