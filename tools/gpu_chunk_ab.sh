#!/usr/bin/env bash
# A/B of the INT8 chunk size (energies per conversion / GEMM launch, RMX_I8_CHUNK) on the darc bench:
# fewer, longer launches amortise the per-chunk stream hand-offs and kernel tails
set -u
mkdir -p gpurun_out
TAG=${1:-ch}
RMX_I8_CHUNK=16 timeout 600 python -m pytest tests/test_rint8.py -q -x -k "darc_block or sweep_parity" > gpurun_out/${TAG}_pytest.log 2>&1
tail -1 gpurun_out/${TAG}_pytest.log
ARGS="--steps 5 --warmup 3 --no-e2e --no-cpu-baseline"
for C in 8 16 24 8 16; do
  RMX_I8_CHUNK=$C timeout 600 python bench.py $ARGS > gpurun_out/${TAG}_c$C.json 2> gpurun_out/${TAG}_c$C.err
  python - "$TAG" "$C" <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/{sys.argv[1]}_c{sys.argv[2]}.json").read().strip().splitlines()[-1])
print("chunk", sys.argv[2], round(d["value"], 1), json.dumps(d.get("kernel_ms")), d["timing"]["runs_ms"], d["clocks"]["sm_mhz"])
PY
done
