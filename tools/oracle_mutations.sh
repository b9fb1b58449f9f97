#!/usr/bin/env bash
# Mutation check of the oracle pins: each plausible mistake (wrong sign of 1/(E_k-E), dropped
# 1/2a, wrong index in aR G'_j, wrong sign of iK, squared row instead of w_i w_j, perturbed
# elimination factor, scaled or mis-indexed sampled R entries) must make tests/test_oracle_pins.py fail. Restores the source after.
set -u
cd "$(dirname "$0")/.."
src=oracle/rmx_oracle.c
cp $src /tmp/rmx_oracle_orig.c
muts=(
 's/d\[k\] = 1.0L \/ diff;/d[k] = -1.0L \/ diff;/'
 's/R\[i \* nch + j\] = s \* inv2a;/R[i * nch + j] = s * inv2a * 2.0L;/'
 's/- aR \* (ld)Gp\[j\];/- aR * (ld)Gp[i];/'
 's/- I \* K\[i \* n + j\];/+ I * K[i * n + j];/'
 's/s += (ld)wi\[k\] \* (ld)wj\[k\] \* d\[k\];/s += (ld)wi[k] * (ld)wi[k] * d[k];/'
 's/ld f = A\[r \* n + c\] \/ piv;/ld f = A[r * n + c] \/ piv * (r == n-1 ? 1.0000001L : 1.0L);/'
 's/out\[p\] = (double)(s \* inv2a);/out[p] = (double)(s * inv2a * 1.001L);/'
 's/const double \*wi = w + ii\[p\] \* ldw, \*wj = w + jj\[p\] \* ldw;/const double *wi = w + ii[p] * ldw, *wj = w + ii[p] * ldw;/'
)
fail=0
for m in "${muts[@]}"; do
  cp /tmp/rmx_oracle_orig.c $src; sed -i "$m" $src
  if cmp -s /tmp/rmx_oracle_orig.c $src; then echo "NOT APPLIED: $m"; fail=1; continue; fi
  if python -m pytest tests/test_oracle_pins.py -q -x >/dev/null 2>&1; then
    echo "SURVIVED: $m"; fail=1
  else
    echo "killed:   $m"
  fi
done
cp /tmp/rmx_oracle_orig.c $src
python -c "import oracle; oracle.build(force=True)"
exit $fail
