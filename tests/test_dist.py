"""Multi-process (world_size 2, gloo, CPU) tests of the energy-sharding plumbing of
paper_1403_5524_b200.dist: block-cyclic partition, W/E_k broadcast from rank 0
("ONLY processor 0 to read, then distribute (i.e. MPI_BCAST)"), and the single
all-gather of per-energy summaries with reassembly in mesh order. The per-rank compute is replaced
by a deterministic function of the energy index (the CUDA sweep itself is covered by the GPU tests);
the N>1 GPU path uses exactly these functions with the nccl backend."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1403_5524_b200 import dist as rdist
import rmx_synth as syn


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, ne, block, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    rdist.init_process_group("gloo")
    try:
        # broadcast of replicated inputs from rank 0
        W = torch.arange(12, dtype=torch.float64).reshape(3, 4) if rank == 0 else torch.zeros(3, 4, dtype=torch.float64)
        Ek = torch.linspace(0, 1, 5, dtype=torch.float64) if rank == 0 else torch.zeros(5, dtype=torch.float64)
        rdist.broadcast_inputs([W, Ek])
        # this rank's shard, processed in order; "summary" = deterministic function of the index
        idx = rdist.shard_indices(ne, block, world, rank)
        local = torch.stack([torch.tensor([float(i), float(i) ** 0.5, -float(i)], dtype=torch.float64)
                             for i in idx]) if len(idx) else torch.zeros((0, 3), dtype=torch.float64)
        full = rdist.gather_summaries(local, ne, block, world)
        out_q.put((rank, W.numpy().copy(), Ek.numpy().copy(), full.numpy().copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("ne,block", [(37, 5), (10, 3), (8, 8), (3, 4)])
def test_gloo_world2_broadcast_and_gather(ne, block):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, ne, block, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    expect = np.stack([[float(i), float(i) ** 0.5, -float(i)] for i in range(ne)])
    for rank, W, Ek, full in res:
        assert np.array_equal(W, np.arange(12, dtype=np.float64).reshape(3, 4))
        assert np.array_equal(Ek, np.linspace(0, 1, 5))
        assert np.array_equal(full, expect), rank


def test_partition_covers_mesh_exactly_once():
    for ne in (1, 7, 100, 1001):
        for block in (1, 3, 296):
            for world in (1, 2, 4, 8):
                all_idx = np.concatenate([rdist.shard_indices(ne, block, world, r) for r in range(world)])
                assert np.array_equal(np.sort(all_idx), np.arange(ne))
                lens = [len(rdist.shard_indices(ne, block, world, r)) for r in range(world)]
                assert max(lens) - min(lens) <= block
                assert rdist.padded_shard_len(ne, block, world) == max(lens)


def test_block_cyclic_balances_darc_cost():
    """contiguous shards are imbalanced (K and T cost grow with n_o(E)); block-cyclic
    dealing balances the cost model to well under 1% at 8 ranks."""
    cfg = syn.CONFIGS["darc"]
    rng = np.random.default_rng(0)
    lev = rng.uniform(0.0, 50.0, 300)  # same recipe as rmx_synth (levels -> thresholds)
    eps = np.sort(np.concatenate([np.repeat(lev[:200], 7), np.repeat(lev[200:], 6)]))
    E = syn.mesh(cfg["lo"], cfg["hi"], cfg["ne"])
    cost = rdist.cost_model(cfg["nch"], cfg["nlev"], syn.n_open(eps, E))
    contiguous = rdist.imbalance(cost, cfg["ne"] // 8, 8)
    assert contiguous > 0.15                               # measured 0.186
    assert rdist.imbalance(cost, 16, 8) < 2e-3             # fine blocks: ~1e-3
    assert rdist.imbalance(cost, 296, 8) < 0.03            # bench batch (2 x 148): 0.0185


def _worker_case(rank, world, port, out_q):
    """bench.py's N > 1 input path: rank 0 generates the case, the other ranks generate nothing and
    receive W, E_k, thresholds and mesh (rdist.broadcast_case); then a bench-style gather of the
    row sums of the blocks each rank processed (explicit shards), reassembled in mesh order."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    rdist.init_process_group("gloo")
    try:
        case = syn.make_case("tiny") if rank == 0 else None
        w, Ek, eps, E, a = rdist.broadcast_case(case, torch.device("cpu"))
        ne, block, steps = len(E), 64, 3
        shards = []
        for r in range(world):  # bench.py timed_shards: `steps` blocks spread over the rank's blocks
            blocks = rdist.cyclic_blocks(ne, block, world, r)
            shards.append(np.concatenate([np.arange(*rdist.block_range(blocks[int((s + 0.5) * len(blocks) / steps)],
                                                                         ne, block)) for s in range(steps)]))
        mine = torch.from_numpy(np.stack([E.numpy()[shards[rank]], -E.numpy()[shards[rank]]], axis=1))
        full = rdist.gather_summaries(mine, ne, block, world, shards)
        out_q.put((rank, w.numpy().copy(), Ek.numpy().copy(), eps.numpy().copy(), E.numpy().copy(), a,
                   full.numpy().copy(), [s.tolist() for s in shards]))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_broadcast_case_and_partial_gather():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_case, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    c = syn.make_case("tiny")
    for rank, w, Ek, eps, E, a, full, shards in res:
        assert w.shape == (c.nch, c.nlev + (c.nlev & 1))
        assert np.array_equal(w[:, :c.nlev], c.w) and np.all(w[:, c.nlev:] == 0)
        assert np.array_equal(Ek, c.Ek) and np.array_equal(eps, c.eps) and np.array_equal(E, c.E)
        assert a == c.a
        covered = np.concatenate([np.array(s) for s in shards])
        assert len(np.unique(covered)) == len(covered)
        expect = np.zeros((len(E), 2))
        expect[covered, 0], expect[covered, 1] = E[covered], -E[covered]
        assert np.array_equal(full, expect), rank


def test_bench_gpus_refuses_without_enough_devices():
    """`python bench.py --gpus N` outside torchrun launches N ranks through torch.distributed.run, and
    refuses with one clear line (exit 2) when fewer than N GPUs are visible."""
    import subprocess
    import sys
    if torch.cuda.is_available() and torch.cuda.device_count() >= 64:
        pytest.skip("box has 64 GPUs")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "64", "--steps", "1"],
                         cwd=root, env=env, capture_output=True, text=True, timeout=300)
    assert out.returncode == 2, out.stdout + out.stderr
    assert "refusing to run 64 ranks" in out.stderr
    # launched with a WORLD_SIZE that disagrees with --gpus: refused as well
    env.update(WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "4", "--steps", "1"],
                         cwd=root, env=env, capture_output=True, text=True, timeout=300)
    assert out.returncode == 2 and "WORLD_SIZE=2" in out.stderr, out.stdout + out.stderr
