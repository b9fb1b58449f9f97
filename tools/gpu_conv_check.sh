#!/usr/bin/env bash
# A/B of the X-residue conversion: tensor-core byte-weight sums (default) vs dp4a (RMX_I8_CONV_ALU):
# INT8 parity tests, then the darc bench under both (kernel breakdown from the instrumented run).
set -u
mkdir -p gpurun_out
TAG=${1:-conv}
timeout 900 python -m pytest tests/test_rint8.py -q -x -rA > gpurun_out/${TAG}_pytest.log 2>&1
tail -3 gpurun_out/${TAG}_pytest.log
ARGS="--steps 5 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 600 python bench.py $ARGS > gpurun_out/${TAG}_tc.json 2> gpurun_out/${TAG}_tc.err
RMX_I8_CONV_ALU=1 timeout 600 python bench.py $ARGS > gpurun_out/${TAG}_alu.json 2> gpurun_out/${TAG}_alu.err
for f in tc alu; do python - "$f" "$TAG" <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/{sys.argv[2]}_{sys.argv[1]}.json").read().strip().splitlines()[-1])
print(sys.argv[1], round(d["value"], 1), d.get("ms_per_step"), json.dumps(d.get("kernel_ms"))[:700], d["timing"]["runs_ms"])
PY
done
