#!/usr/bin/env bash
# A/B of the paired tile-row order of the CTA GEMM's C -= A.B (librmx.so) against the row-major
# order everywhere (librmx_np.so, -DRMX_NO_TILE_PAIRS): K parity subset, then darc bench lines
# alternating the two libraries
set -u
mkdir -p gpurun_out
TAG=${1:-tp}
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/${TAG}_pytest.log 2>&1
tail -1 gpurun_out/${TAG}_pytest.log
ARGS="--steps 5 --warmup 3 --no-e2e --no-cpu-baseline"
for v in pairs np pairs np; do
  if [ $v = np ]; then export RMX_LIB=paper_1403_5524_b200/librmx_np.so; else unset RMX_LIB; fi
  timeout 600 python bench.py $ARGS > gpurun_out/${TAG}_$v.json 2> gpurun_out/${TAG}_$v.err
  python - "$TAG" "$v" <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/{sys.argv[1]}_{sys.argv[2]}.json").read().strip().splitlines()[-1])
print(sys.argv[2], round(d["value"], 1), json.dumps(d.get("kernel_ms")), d["timing"]["runs_ms"], d["clocks"]["sm_mhz"])
PY
done
unset RMX_LIB
ARGS1="--steps 1 --warmup 3 --no-e2e --no-cpu-baseline --repeats 1"
ncu --set full --import-source on --clock-control none -k regex:match_kernel -s 3 -c 1 \
    -o gpurun_out/${TAG}_match python bench.py $ARGS1 > gpurun_out/${TAG}_ncu_match.log 2>&1
echo "ncu rc=$?"
