#!/usr/bin/env bash
# A/B of the tensor-core conversion's elements per thread (RMX_I8_CONV_EL 8 / 4): bitwise test, ncu of
# one launch each, darc bench lines
set -u
mkdir -p gpurun_out
TAG=${1:-el}
timeout 600 python -m pytest tests/test_rint8.py -q -x -k "tc_conversion" > gpurun_out/${TAG}_pytest.log 2>&1
tail -1 gpurun_out/${TAG}_pytest.log
ARGS="--steps 1 --warmup 3 --no-e2e --no-cpu-baseline --repeats 1"
for EL in 4 8; do
  RMX_I8_CONV_EL=$EL ncu --set full --import-source on --clock-control none -k regex:oz_convert -s 12 -c 1 \
      -o gpurun_out/${TAG}_el$EL python bench.py $ARGS > gpurun_out/${TAG}_ncu_el$EL.log 2>&1
  echo "ncu el$EL rc=$?"
done
for EL in 4 8; do
  RMX_I8_CONV_EL=$EL timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_b$EL.json 2> gpurun_out/${TAG}_b$EL.err
  python - "$TAG" "$EL" <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/{sys.argv[1]}_b{sys.argv[2]}.json").read().strip().splitlines()[-1])
print("el", sys.argv[2], round(d["value"], 1), json.dumps(d.get("kernel_ms")), d["timing"]["runs_ms"], d["clocks"]["sm_mhz"])
PY
done
