#!/usr/bin/env bash
# Mutation check of the oracle pins of the SURVEY §8(f) rows (NEXT-1 photoionisation, NEXT-2 level-pair
# collision strengths, NEXT-4 convolution / Maxwell average): each plausible mistake must make the CPU
# pins of tests/test_photo.py, tests/test_levels.py or tests/test_post.py fail. Restores the sources.
set -u
cd "$(dirname "$0")/.."
csrc=oracle/rmx_oracle.c
psrc=oracle/__init__.py
cp $csrc /tmp/rmx_oracle_orig_n.c
cp $psrc /tmp/oracle_init_orig_n.py
cmuts=(
 's/s += (ld)w\[i \* ldw + k\] \* ((ld)d\[k\] \/ ((ld)Ek\[k\] - (ld)E));/s += (ld)w[i * ldw + k] * ((ld)d[k] \/ ((ld)E - (ld)Ek[k]));/'
 's/M\[j\] = 0.5L \* s; /M[j] = s; /'
 's/- I \* (ld)K\[j \* n + l\];/+ I * (ld)K[j * n + l];/'
 's/ld s = g\[j\] \* (ld)Fp\[j\];/ld s = 0.0L;/'
 's/s += g\[i\] \* (ld)Gp\[i\] \* (ld)K\[i \* n + j\];/s += g[i] * (ld)Gp[i] * (ld)K[j * n + i] * (i == 0 ? 1.001L : 1.0L);/'
)
pmuts=(
 's/acc = T2l\[ls\[la\]:ls\[la + 1\], ls\[lb\]:ls\[lb + 1\]\].sum()/acc = T2l[ls[la]:ls[la + 1], ls[la]:ls[la + 1]].sum()/'
 's/om\[la, lb\] = float(np.longdouble(g) \* acc)/om[la, lb] = float(acc)/'
 's/if ls\[lb + 1\] > n_open:/if ls[lb + 1] > n_open + 1:/'
 's/out\[m, i\] = float((gw \* xb\[lo:hi + 1\]).sum() \/ gw.sum())/out[m, i] = float((gw * xb[lo:hi + 1]).sum() \/ g.sum())/'
 's/M = int(np.floor(5.0 \* s \/ dE))/M = int(np.floor(5.0 * s \/ dE)) + 1/'
 's/x.astype(np.longdouble)).sum(axis=0) \/ c.sum()\]/x.astype(np.longdouble)).sum(axis=0)]/'
 's/side="right"/side="left"/'
 's/np.exp(-(E\[first:\] - np.longdouble(Eth\[p\])) \/ kt) \/ kt/np.exp(-(E[first:] - np.longdouble(Eth[p])) \/ kt)/'
)
TESTS="tests/test_photo.py tests/test_levels.py tests/test_post.py"
fail=0
run() {  # $1 = description
  if python -m pytest $TESTS -q -x -m "not gpu" >/dev/null 2>&1; then echo "SURVIVED: $1"; fail=1; else echo "killed:   $1"; fi
}
for m in "${cmuts[@]}"; do
  cp /tmp/rmx_oracle_orig_n.c $csrc; sed -i "$m" $csrc
  if cmp -s /tmp/rmx_oracle_orig_n.c $csrc; then echo "NOT APPLIED: $m"; fail=1; continue; fi
  python -c "import oracle; oracle.build(force=True)" >/dev/null 2>&1
  run "$m"
done
cp /tmp/rmx_oracle_orig_n.c $csrc
python -c "import oracle; oracle.build(force=True)" >/dev/null 2>&1
for m in "${pmuts[@]}"; do
  cp /tmp/oracle_init_orig_n.py $psrc; sed -i "$m" $psrc
  if cmp -s /tmp/oracle_init_orig_n.py $psrc; then echo "NOT APPLIED: $m"; fail=1; continue; fi
  run "$m"
done
cp /tmp/oracle_init_orig_n.py $psrc
exit $fail
