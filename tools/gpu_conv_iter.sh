#!/usr/bin/env bash
# one iteration on the conversion kernel: bitwise test, ncu of one launch, darc bench line
set -u
mkdir -p gpurun_out
TAG=${1:-conv}
timeout 600 python -m pytest tests/test_rint8.py -q -x -k "tc_conversion or darc_block" > gpurun_out/${TAG}_pytest.log 2>&1
tail -1 gpurun_out/${TAG}_pytest.log
ARGS="--steps 1 --warmup 3 --no-e2e --no-cpu-baseline --repeats 1"
ncu --set full --import-source on --clock-control none -k regex:oz_convert -s 12 -c 1 \
    -o gpurun_out/${TAG}_tc python bench.py $ARGS > gpurun_out/${TAG}_ncu_tc.log 2>&1
echo "ncu rc=$?"
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
python - "$TAG" <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/{sys.argv[1]}_bench.json").read().strip().splitlines()[-1])
print(round(d["value"], 1), d.get("ms_per_step"), json.dumps(d.get("kernel_ms")), d["timing"]["runs_ms"])
PY
