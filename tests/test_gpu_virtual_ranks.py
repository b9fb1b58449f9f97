"""Bitwise determinism across GPU counts (per-energy outputs identical at P = 1, 2,
4, 8; Table 1 runs one energy mesh on 1024-8192 cores). On one GPU, P virtual ranks
run their block-cyclic shards one after the other exactly as bench.py's ranks would (each rank sweeps
its own blocks in order, batch = the block size), the row sums are reassembled in mesh order by the
same index arithmetic as paper_1403_5524_b200.dist.gather_summaries, and must equal the P = 1 sweep
bit for bit - for both R formations (the INT8-CRT chunking of 8..64 energies follows the batch, so
this also checks that an energy's arithmetic does not depend on which energies share its chunk)."""
import numpy as np
import pytest

import rmx_synth as syn
from paper_1403_5524_b200 import dist as rdist

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("algo", ["int8", "dmma"])
def test_virtual_ranks_bitwise(algo):
    import torch
    import paper_1403_5524_b200 as rmx
    ctx = rmx.Context()
    ctx.set_r_algo(rmx.R_INT8 if algo == "int8" else rmx.R_DMMA)
    # nch >= 256 so R_INT8 really runs the CRT path; closed channels; 296-energy mesh, blocks of 24
    c = syn.brute_force_case(300, 1200, 21, ne=296, lo=0.5, hi=9.0, a=12.0, eps_hi=4.0)
    F, G, Fp, Gp = syn.asymptotic(c.eps, c.E, c.a)
    no = syn.n_open(c.eps, c.E)
    ne, block = c.ne, 24
    ref = ctx.sweep(c.w, c.Ek, c.a, c.E, F, G, Fp, Gp, no, batch=block)
    torch.cuda.synchronize()
    rs1, st1 = ref["rowsum"].cpu().numpy(), ref["status"].cpu().numpy()
    assert np.all(st1 == 0)
    for P in (2, 4, 8):
        full = np.full_like(rs1, np.nan)
        for r in range(P):
            idx = rdist.shard_indices(ne, block, P, r)
            if len(idx) == 0:
                continue
            out = ctx.sweep(c.w, c.Ek, c.a, c.E[idx], F[idx], G[idx], Fp[idx], Gp[idx], no[idx], batch=block)
            torch.cuda.synchronize()
            assert np.all(out["status"].cpu().numpy() == 0)
            full[idx] = out["rowsum"].cpu().numpy()
        assert np.array_equal(full, rs1), (algo, P)
    # other batch sizes on the whole mesh: 296 (one INT8 launch set), 37, 8 (the minimum INT8 chunk)
    for batch in (296, 37, 8):
        out = ctx.sweep(c.w, c.Ek, c.a, c.E, F, G, Fp, Gp, no, batch=batch)
        torch.cuda.synchronize()
        assert np.array_equal(out["rowsum"].cpu().numpy(), rs1), (algo, batch)
