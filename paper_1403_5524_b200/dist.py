"""Multi-GPU plumbing for the energy sweep: one process per GPU, energies
sharded block-cyclically, W and E_k replicated by one broadcast from rank 0 (the analog of the
paper's "ONLY processor 0 to read, then distribute (i.e. MPI_BCAST)", §3 item 1),
and the per-energy summaries returned by one all-gather. Nothing here computes the method: the
per-rank work is ``Context.sweep`` (librmx). The functions are device-agnostic so the partition,
broadcast and reassembly logic is tested with the gloo backend on CPU (tests/test_dist.py).

Energies are independent (no exchange inside the hot loop), so the hot path has no collective;
block-cyclic dealing balances the n_open-dependent cost of K and T across ranks.
"""
from __future__ import annotations

import os
from typing import List, Optional, Tuple

import numpy as np


def env_rank_world() -> Tuple[int, int, int]:
    """(rank, world_size, local_rank) from the torchrun environment (defaults: single process)."""
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def n_blocks(ne: int, block: int) -> int:
    return (ne + block - 1) // block


def cyclic_blocks(ne: int, block: int, world: int, rank: int) -> List[int]:
    """Block indices owned by `rank`: blocks of `block` consecutive energies dealt round-robin."""
    return list(range(rank, n_blocks(ne, block), world))


def block_range(b: int, ne: int, block: int) -> Tuple[int, int]:
    lo = b * block
    return lo, min(ne, lo + block)


def shard_indices(ne: int, block: int, world: int, rank: int) -> np.ndarray:
    """Mesh indices of this rank's shard, in processing order."""
    out = [np.arange(*block_range(b, ne, block)) for b in cyclic_blocks(ne, block, world, rank)]
    return np.concatenate(out) if out else np.zeros(0, dtype=np.int64)


def padded_shard_len(ne: int, block: int, world: int) -> int:
    """Equal per-rank length for the all-gather (every shard padded to the longest)."""
    return max(len(shard_indices(ne, block, world, r)) for r in range(world))


def broadcast_inputs(tensors, src: int = 0):
    """Broadcast each tensor in place from `src` (W, E_k ...). Shapes/dtypes must already agree."""
    import torch.distributed as dist
    for t in tensors:
        dist.broadcast(t, src=src)
    return tensors


def gather_summaries(local: "torch.Tensor", ne: int, block: int, world: int, shards=None):
    """All-gather per-energy summaries [n_local, ...] from every rank (single collective) and
    reassemble them into mesh order [ne, ...] on every rank. shards[r] = the mesh indices rank r
    processed, in its processing order (default: its whole block-cyclic shard, shard_indices);
    mesh points no rank processed are left zero."""
    import torch
    import torch.distributed as dist
    if shards is None:
        shards = [shard_indices(ne, block, world, r) for r in range(world)]
    L = max(len(s) for s in shards)
    tail = tuple(local.shape[1:])
    assert local.shape[0] == len(shards[dist.get_rank()])
    pad = torch.zeros((L,) + tail, dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    out = torch.empty((world * L,) + tail, dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(out, pad)
    full = torch.zeros((ne,) + tail, dtype=local.dtype, device=local.device)
    for r in range(world):
        idx = np.asarray(shards[r], dtype=np.int64)
        if len(idx):
            full[torch.from_numpy(idx).to(local.device)] = out[r * L: r * L + len(idx)]
    return full


def broadcast_case(case, device, src: int = 0):
    """The replicated inputs of the sweep from rank `src` (the paper's root read + MPI_BCAST,
    PAPER.md:208-211): rank src passes the generated rmx_synth.Case, the other ranks pass None and
    generate nothing. Returns (w [nch, ldw] (ldw even, zero padded), Ek [nlev], eps [nch],
    E [ne] (float64 tensors on `device`), a) on every rank: one small header broadcast, then one
    broadcast per array."""
    import torch
    import torch.distributed as dist
    rank = dist.get_rank()
    hdr = torch.zeros(4, dtype=torch.float64, device=device)
    if rank == src:
        hdr[:] = torch.tensor([case.nch, case.nlev, case.ne, case.a], dtype=torch.float64)
    dist.broadcast(hdr, src=src)
    nch, nlev, ne, a = int(hdr[0]), int(hdr[1]), int(hdr[2]), float(hdr[3])
    ldw = nlev + (nlev & 1)
    w = torch.zeros((nch, ldw), dtype=torch.float64, device=device)
    Ek = torch.empty(nlev, dtype=torch.float64, device=device)
    eps = torch.empty(nch, dtype=torch.float64, device=device)
    E = torch.empty(ne, dtype=torch.float64, device=device)
    if rank == src:
        w[:, :nlev] = torch.from_numpy(case.w).to(device)
        Ek.copy_(torch.from_numpy(case.Ek))
        eps.copy_(torch.from_numpy(case.eps))
        E.copy_(torch.from_numpy(case.E))
    broadcast_inputs([w, Ek, eps, E], src=src)
    return w, Ek, eps, E, a


def imbalance(costs: np.ndarray, block: int, world: int) -> float:
    """max/mean - 1 of per-rank total cost under block-cyclic dealing."""
    ne = len(costs)
    per = [costs[shard_indices(ne, block, world, r)].sum() for r in range(world)]
    return float(max(per) / (np.mean(per) if np.mean(per) > 0 else 1.0) - 1.0)


def cost_model(nch: int, nlev: int, n_open: np.ndarray) -> np.ndarray:
    """Algorithmic flops per energy: F_R + F_K + F_T."""
    no = n_open.astype(np.float64)
    return nch * (nch + 1.0) * nlev + (2.0 / 3.0) * nch ** 3 + 2.0 * nch ** 2 * no + (16.0 / 3.0) * no ** 3


def init_process_group(backend: Optional[str] = None, timeout_s: float = 600.0):
    """torch.distributed init from the torchrun env (127.0.0.1 rendezvous by default). A collective
    that does not complete within timeout_s raises on every rank instead of hanging (NCCL async error
    handling on: the watchdog aborts the communicator and the process exits non-zero)."""
    import datetime
    import torch.distributed as dist
    if dist.is_initialized():
        return
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29511")
    os.environ.setdefault("TORCH_NCCL_ASYNC_ERROR_HANDLING", "1")
    if backend is None:
        import torch
        backend = "nccl" if torch.cuda.is_available() else "gloo"
    kw = {}
    if backend == "nccl":
        import torch
        kw["device_id"] = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    dist.init_process_group(backend=backend, timeout=datetime.timedelta(seconds=timeout_s), **kw)
