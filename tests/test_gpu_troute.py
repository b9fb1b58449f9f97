"""The T route of rmx_collision_strength (S5, reading T2: T = 2(A^-1 - I), A = I - iK_oo,
complex-symmetric LDL^T without pivoting, 3M complex GEMMs) against the oracle's pivoted complex
elimination in long double (oracle_T2, BASELINE.json:5 T = 2iK(I - iK)^-1) on given K matrices:

* open-block sizes at and around every blocking boundary of the route (64-wide diagonal blocks,
  128-row Z block rows, 256-column outer blocks, 128 x 32 / 128 x 64 GEMM tiles), plus closed rows and
  columns around the open block that must be ignored;
* conditioning far beyond the darc samples: a rank-1 (and a two-opposite-sign rank-2) term of size
  lambda = 1e2 .. 1e8 on top of an O(1) symmetric K - the regime where round 1's SPD route through
  I + K^2 lost (u lambda^2) and the complex route must stay at ~u lambda (1e-8 is reached at
  lambda ~ 1e8 only by a factor-100 margin);
* bitwise symmetry of |T|^2, the row-sum identity's bounds 0 <= sum_j |T_ij|^2 <= 4.
"""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


def nrel(x, ref):
    den = np.max(np.abs(ref))
    return float(np.max(np.abs(x - ref)) / (den if den > 0 else 1.0))


def make_K(o, nc, lam, kind, seed):
    rng = np.random.default_rng(seed)
    n = o + nc
    K = rng.normal(0.0, 1.0, (n, n))
    K = 0.5 * (K + K.T)
    if lam > 0 and o > 1:
        q = np.linalg.qr(rng.normal(size=(o, 2)))[0]
        K[:o, :o] += lam * np.outer(q[:, 0], q[:, 0])
        if kind == "rank2":
            K[:o, :o] -= lam * np.outer(q[:, 1], q[:, 1])
    K[:o, :o] = 0.5 * (K[:o, :o] + K[:o, :o].T)  # exactly symmetric open block (reading M1)
    return K


CASES = [(o, 0.0, "rank1") for o in (1, 2, 63, 64, 65, 127, 128, 129, 191, 255, 256, 257, 320, 513)]
CASES += [(o, lam, kind) for o in (65, 257) for lam in (1e2, 1e5, 1e8) for kind in ("rank1", "rank2")]


@pytest.fixture(scope="module")
def ctx():
    import paper_1403_5524_b200 as rmx
    return rmx.Context()


@pytest.mark.parametrize("o,lam,kind", CASES)
def test_t_route_against_oracle(ctx, o, lam, kind):
    import torch
    nc = 7
    K = make_K(o, nc, lam, kind, seed=o + int(np.log10(lam + 1)))
    n = o + nc
    Ks = np.stack([K, K])
    no = np.array([o, o], dtype=np.int32)
    T2, rs, st = ctx.collision_strength(torch.from_numpy(Ks), no)
    torch.cuda.synchronize()
    T2, rs, st = T2.cpu().numpy(), rs.cpu().numpy(), st.cpu().numpy()
    assert np.all(st == 0)
    assert np.array_equal(T2[0], T2[1])  # per-energy arithmetic independent of the slot
    ref_t2, ref_rs, _, _, unit, rst = oracle.T2(K, o)
    assert rst == 0 and unit < 1e-12
    e_t, e_r = nrel(T2[0], ref_t2), nrel(rs[0], ref_rs)
    assert e_t < 1e-8 and e_r < 1e-8, (o, lam, kind, e_t, e_r)
    assert np.array_equal(T2[0], T2[0].T)
    assert np.all(T2[0][o:, :] == 0) and np.all(T2[0][:, o:] == 0)
    assert np.all(rs[0] >= 0) and np.all(rs[0] <= 4.0 * (1 + 1e-12))
    # the error scales like u lambda (<= 45 u lambda + 1e-12), not like round 1's u lambda^2
    assert e_t < 5e-15 * max(1.0, lam) + 1e-12, (o, lam, e_t)
