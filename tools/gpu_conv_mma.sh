#!/usr/bin/env bash
# A/B of the X-residue conversion variants: tensor-core (default), warp-level IMMA with 2 / 3 CTAs
# per SM (RMX_I8_CONV_MMA=2|3): bitwise test, ncu of one launch each, darc bench lines
set -u
mkdir -p gpurun_out
TAG=${1:-mma}
timeout 600 python -m pytest tests/test_rint8.py -q -x -k "tc_conversion" > gpurun_out/${TAG}_pytest.log 2>&1
tail -1 gpurun_out/${TAG}_pytest.log
ARGS="--steps 1 --warmup 3 --no-e2e --no-cpu-baseline --repeats 1"
for V in 2 3; do
  RMX_I8_CONV_MMA=$V ncu --set full --import-source on --clock-control none -k regex:oz_convert -s 12 -c 1 \
      -o gpurun_out/${TAG}_m$V python bench.py $ARGS > gpurun_out/${TAG}_ncu_m$V.log 2>&1
  echo "ncu m$V rc=$?"
done
for V in tc 2 3; do
  if [ $V = tc ]; then unset RMX_I8_CONV_MMA; else export RMX_I8_CONV_MMA=$V; fi
  timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_b$V.json 2> gpurun_out/${TAG}_b$V.err
  python - "$TAG" "$V" <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/{sys.argv[1]}_b{sys.argv[2]}.json").read().strip().splitlines()[-1])
print("conv", sys.argv[2], round(d["value"], 1), json.dumps(d.get("kernel_ms")), d["timing"]["runs_ms"], d["clocks"]["sm_mhz"])
PY
done
