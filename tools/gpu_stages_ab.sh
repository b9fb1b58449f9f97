#!/usr/bin/env bash
# A/B of the pair-GEMM ring depth (RMX_I8_STAGES 7 / 6 / 5: room for 0 / 1 / 2 conversion CTAs beside
# a GEMM CTA) on the darc bench, tensor-core conversion
set -u
mkdir -p gpurun_out
TAG=${1:-stg}
timeout 600 python -m pytest tests/test_rint8.py -q -x -k "tc_conversion or darc_block or sweep_parity" > gpurun_out/${TAG}_pytest.log 2>&1
tail -1 gpurun_out/${TAG}_pytest.log
for S in 7 6 5; do
  RMX_I8_STAGES=$S timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_s$S.json 2> gpurun_out/${TAG}_s$S.err
  python - "$TAG" "$S" <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/{sys.argv[1]}_s{sys.argv[2]}.json").read().strip().splitlines()[-1])
print("stages", sys.argv[2], round(d["value"], 1), json.dumps(d.get("kernel_ms")), d["timing"]["runs_ms"], d["clocks"]["sm_mhz"])
PY
done
