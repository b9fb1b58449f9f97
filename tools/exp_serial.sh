set -u
mkdir -p gpurun_out
for v in 0 1 0 1; do
  if [ $v = 1 ]; then export RMX_I8_SERIAL=1; else unset RMX_I8_SERIAL; fi
  timeout 600 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('serial=$v', round(d['value'],2), d.get('kernel_ms'), d['clocks']['sm_mhz'])"
done
