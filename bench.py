#!/usr/bin/env python
"""Bench: energies/s of the full R -> K -> |T|^2 sweep (BASELINE.json:2 metric) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config darc] [--impl reference]
    torchrun --nproc-per-node N --master-addr 127.0.0.1 ... bench.py --gpus N ...

A step = one rmx_sweep call (R formation, matching, T epilogue) over one batch of energies of the
workload's mesh (default: BASELINE.json:10 'darc', nch=2000, nlev=40000, the configuration the
north_star target is quoted on; it fits one GPU). Energy batches are dealt block-cyclically to the
ranks (no collective inside the timed region; scaling "weak": fixed energies per GPU per step).
value  = energies processed by all ranks / max-over-ranks device time (CUDA events, inputs in HBM)
e2e    = same metric through rmx_sweep_host: host (pinned) inputs -> device -> host row sums
roofline: dominant kernel = R formation, FP64 DMMA, algorithmic flops nch(nch+1)nlev per energy
cpu_baseline: the CPU oracle (oracle/) on a bounded sample (rank 0, N = 1 only)
--impl reference: the oracle itself as the reference arm (PAPER has no runnable reference code).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import rmx_synth as syn  # noqa: E402
from paper_1403_5524_b200 import dist as rdist  # noqa: E402

# FP64 DMMA peak measured on this pool's B200 by tools/fp64_peak.cu (profiles/r01_fp64_peak.jsonl);
# MEASURED_PEAKS.json carries no FP64 entry and B200_PROFILING.md states no FP64 fallback.
FP64_DMMA_PEAK_TFLOPS = 37.1
FP64_DFMA_PEAK_TFLOPS = 34.2


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except (OSError, ValueError):
        return {}


def ncu_traffic(workload: str, batch: int, kernel: str = "rform"):
    """DRAM bytes (read + write) per launch of the dominant kernel from the newest committed full ncu
    capture (profiles/rNN_ncu_kernels.json, written by tools/summarize_profiles.py), when that
    capture was taken on the same workload and energies per launch; else None. Several captured
    kernels matching `kernel` in one capture are summed."""
    import glob
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_ncu_kernels.json")), reverse=True):
        try:
            d = json.load(open(path))
        except (OSError, ValueError):
            continue
        tot, hit = 0.0, False
        dur = 0.0
        for name, ent in d.items():
            if kernel not in name:
                continue
            wl = ent.get("workload", {})
            rd, wr = ent.get("dram__bytes_read.bytes"), ent.get("dram__bytes_write.bytes")
            if wl.get("config") == workload and wl.get("energies_per_launch") == batch and rd and wr:
                tot += rd + wr
                dur += ent.get("gpu__time_duration.sum") or 0.0
                hit = True
        if hit:
            ncu_traffic.duration_ms = dur  # the captured launch's own (cold, serialised) duration
            return tot, os.path.basename(path)
    return None, None


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--config", default="darc", choices=list(syn.CONFIGS))
    p.add_argument("--batch", type=int, default=0, help="energies per step (0: library default)")
    p.add_argument("--impl", default="rmx", choices=["rmx", "reference"])
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--oracle-sample", type=int, default=1, help="energies in the oracle sample")
    p.add_argument("--repeats", type=int, default=3, help="timed runs of K steps; value = their median")
    p.add_argument("--r-algo", default="int8", choices=["dmma", "int8"],
                   help="R formation: exact CRT on the INT8 tensor cores (default, rint8.cu) or the FP64 DMMA "
                        "contraction (rform.cu)")
    return p.parse_args()


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region (B200_PROFILING.md)."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        self.f.flush()
        self.f.seek(0)
        rows = [r.split(",") for r in self.f.read().strip().splitlines() if r.strip()]
        os.unlink(self.f.name)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in rows if r[0].strip().replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in rows:
            for k, name in enumerate(names):
                if len(r) > 4 + k and "Active" in r[4 + k] and "Not" not in r[4 + k]:
                    reasons.add(name)
        load = [s for s in sm if s > 0.5 * (max(mx) if mx else 1)] or sm
        return {"sm_mhz": statistics.median(load) if load else None,
                "sm_max_mhz": max(mx) if mx else None, "samples": len(rows),
                "reasons": sorted(reasons)}


def oracle_baseline(case, idx, threads):
    """Time the CPU oracle (as it stands) on mesh indices idx; returns (energies/s, seconds)."""
    import oracle
    E = case.E[idx]
    F, G, Fp, Gp = syn.asymptotic(case.eps, E, case.a)
    no = syn.n_open(case.eps, E)
    oracle.build()
    t0 = time.perf_counter()
    out = oracle.sweep(case.w, case.Ek, case.a, E, F, G, Fp, Gp, no, np.arange(len(idx)),
                       want=("rowsum",), threads=threads)
    dt = time.perf_counter() - t0
    assert np.all(out["status"] == 0)
    return len(idx) / dt, dt


def flops_per_energy(nch, nlev, n_open):
    no = np.asarray(n_open, dtype=np.float64)
    fr = nch * (nch + 1.0) * nlev
    fk = (2.0 / 3.0) * nch ** 3 + 2.0 * nch ** 2 * no
    ft = (16.0 / 3.0) * no ** 3
    return fr, fk, ft


def run_reference(args, rank):
    if rank != 0:
        return
    case = syn.make_case(args.config)
    threads = os.cpu_count() or 1
    sample = [case.ne // 2 + s for s in range(max(1, args.oracle_sample))]
    for _ in range(args.warmup):
        oracle_baseline(case, sample, threads)
    times = []
    for _ in range(args.steps):
        _, dt = oracle_baseline(case, sample, threads)
        times.append(dt)
    tot = sum(times)
    v = len(sample) * args.steps / tot
    line = {
        "impl": "reference", "metric": "energies/sec (R->K->|T|^2 sweep)", "value": v,
        "unit": "energies/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * tot / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64 (oracle: long double)", "data": "synthetic (rmx_synth, seed 0)",
        "config": {"workload": args.config, **{k: v2 for k, v2 in syn.CONFIGS[args.config].items()}},
        "cpu_baseline": {"value": v, "unit": "energies/s", "cores": threads, "kind": "oracle",
                         "sample": f"{len(sample)} energy(ies) at mesh index {sample[0]} of {args.config} per step"},
        "e2e": {"value": v, "unit": "energies/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def spawn_ranks(args) -> int:
    """`python bench.py --gpus N` outside torchrun: start N ranks (one process per GPU) with
    torch.distributed.run on this node, 127.0.0.1 rendezvous; refuse if fewer GPUs are visible."""
    import socket
    import torch
    have = torch.cuda.device_count()
    if args.gpus > have:
        print(f"bench.py: --gpus {args.gpus} but only {have} CUDA device(s) visible; "
              f"refusing to run {args.gpus} ranks", file=sys.stderr, flush=True)
        return 2
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    args = parse()
    rank, world, local = rdist.env_rank_world()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(spawn_ranks(args))
    if "WORLD_SIZE" in os.environ and world != args.gpus:
        print(f"bench.py: launched with WORLD_SIZE={world} but --gpus {args.gpus}", file=sys.stderr)
        sys.exit(2)
    if args.impl == "reference":
        run_reference(args, rank)
        return
    import torch
    import paper_1403_5524_b200 as rmx
    torch.cuda.set_device(local)
    if world > 1:
        rdist.init_process_group("nccl")
        print(f"[bench rank {rank}] NCCL communicator: {torch.distributed.get_world_size()} ranks, "
              f"backend {torch.distributed.get_backend()}, device cuda:{local}", file=sys.stderr, flush=True)
    dev = torch.device(f"cuda:{local}")
    cfg = syn.CONFIGS[args.config]
    nch, nlev = cfg["nch"], cfg["nlev"]

    # ---- inputs: rank 0 generates the case (seeded); the other ranks generate nothing and receive
    # W, E_k, the thresholds and the mesh by broadcast (PAPER.md:208-211 root read + MPI_BCAST)
    t_setup = time.perf_counter()
    ldw = nlev + (nlev & 1)
    if world == 1:
        case = syn.make_case(args.config)
        w_d = torch.zeros((nch, ldw), dtype=torch.float64, device=dev)
        w_d[:, :nlev] = torch.from_numpy(case.w).to(dev)
        Ek_d = torch.from_numpy(case.Ek).to(dev)
        eps, E_mesh, a = case.eps, case.E, case.a
    else:
        torch.cuda.synchronize()
        b0 = time.perf_counter()
        w_d, Ek_d, eps_d, E_d, a = rdist.broadcast_case(syn.make_case(args.config) if rank == 0 else None, dev)
        torch.cuda.synchronize()
        bcast_s = time.perf_counter() - b0
        eps, E_mesh = eps_d.cpu().numpy(), E_d.cpu().numpy()
    ctx = rmx.Context(local)
    if args.r_algo == "int8":
        ctx.set_r_algo(rmx.R_INT8)
    ne = len(E_mesh)
    batch = args.batch if args.batch > 0 else 2 * torch.cuda.get_device_properties(dev).multi_processor_count
    if args.config in ("tiny", "small") and args.batch <= 0:
        batch = min(ne, 4096 if args.config == "small" else ne)
    nb = rdist.n_blocks(ne, batch)
    my_blocks = rdist.cyclic_blocks(ne, batch, world, rank)
    nsteps = args.warmup + args.steps

    # The K timed steps walk this rank's blocks spread evenly over the whole mesh (timed step t takes
    # the block at quantile (t + 0.5)/K), so a short run sees the same mix of open-channel counts
    # n_o(E) - and so of matching / T cost - as the full sweep; warm-up step w repeats timed block
    # w mod K (warm-up must not take blocks out of the timed mix).
    def timed_block(blocks, t):
        return blocks[min(len(blocks) - 1, int((t + 0.5) * len(blocks) / args.steps))]

    def block_of_step(s):
        return timed_block(my_blocks, (s % args.steps) if s < args.warmup else s - args.warmup)

    step_inputs = []
    for s in range(nsteps):
        lo, hi = rdist.block_range(block_of_step(s), ne, batch)
        E = E_mesh[lo:hi]
        F, G, Fp, Gp = syn.asymptotic(eps, E, a)
        no = syn.n_open(eps, E)
        step_inputs.append(dict(
            E=torch.from_numpy(E).to(dev), F=torch.from_numpy(F).to(dev), G=torch.from_numpy(G).to(dev),
            Fp=torch.from_numpy(Fp).to(dev), Gp=torch.from_numpy(Gp).to(dev),
            no=torch.from_numpy(no).to(dev), no_host=no, lo=lo, hi=hi))
    setup_s = time.perf_counter() - t_setup

    def one_step(s):
        d = step_inputs[s]
        return ctx.sweep(w_d, Ek_d, a, d["E"], d["F"], d["G"], d["Fp"], d["Gp"], d["no"],
                         batch=batch, prepared=(nlev, ldw))

    # mesh indices each rank processes in the timed region (same block_of_step rule on every rank)
    def timed_shards():
        out = []
        for r in range(world):
            blocks = rdist.cyclic_blocks(ne, batch, world, r)
            idx = [np.arange(*rdist.block_range(timed_block(blocks, t), ne, batch)) for t in range(args.steps)]
            out.append(np.concatenate(idx))
        return out
    shards = timed_shards() if world > 1 else None

    # ---- device-resident timed region -------------------------------------------------------
    for s in range(args.warmup):
        one_step(s)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    stream = torch.cuda.current_stream()

    def timed_region(instrumented):
        """K steps (+ the gather when N > 1) between CUDA events on torch's stream, bracketed by a
        barrier and synchronize on both sides; returns (max-over-ranks ms, outputs)."""
        ctx.set_timing(instrumented)
        ctx.reset_stats()
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        outs_ = []
        ev0.record(stream)
        for s in range(args.warmup, nsteps):
            outs_.append(one_step(s))
        full_ = None
        if world > 1:
            # S6: one all-gather of the per-energy row sums, reassembled in mesh order on every rank,
            # inside the timed wall (first batch launch to gather completion)
            full_ = rdist.gather_summaries(torch.cat([o["rowsum"] for o in outs_]), ne, batch, world, shards)
        ev1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        ms_ = ev0.elapsed_time(ev1)
        if world > 1:
            t = torch.tensor([ms_], dtype=torch.float64, device=dev)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            ms_ = float(t[0])
        return ms_, outs_, full_

    # the median of 3 uninstrumented runs of the K steps is the reported value; a 4th
    # run with per-launch CUDA events (librmx instrumentation, rmx_set_timing) gives the per-kernel
    # breakdown and the roofline's achieved rate (reported separately, never mixed into `value`)
    runs_ms = []
    with ClockSampler(local) as clk:
        for _ in range(args.repeats):
            ms_run, outs, full = timed_region(False)
            runs_ms.append(ms_run)
        ms_instr, outs_i, _ = timed_region(True)
    stats = ctx.stats()
    ctx.set_timing(False)
    ms_max = statistics.median(runs_ms)
    n_energies_local = sum(step_inputs[s]["hi"] - step_inputs[s]["lo"] for s in range(args.warmup, nsteps))
    bad = sum(int((o["status"] != 0).sum()) for o in outs)
    if world > 1:
        t = torch.tensor([float(n_energies_local)], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.SUM)
        n_energies = int(t[0])
    else:
        n_energies = n_energies_local
    ms = ms_max
    value = n_energies / (ms_max / 1e3)

    # ---- roofline of the dominant kernel (R formation) ---------------------------------------
    ms_r, n_r = stats["rform"]
    fr, fk, ft = 0.0, 0.0, 0.0
    for s in range(args.warmup, nsteps):
        f_r, f_k, f_t = flops_per_energy(nch, nlev, step_inputs[s]["no_host"])
        fr += float(np.sum(np.broadcast_to(f_r, step_inputs[s]["no_host"].shape)))
        fk += float(np.sum(f_k))
        ft += float(np.sum(f_t))
    achieved_r = fr / (ms_r / 1e3) / 1e12 if ms_r > 0 else None
    # ---- the per-energy dense LA kernels (matching, T epilogue): executed algorithmic flops of the
    # routes in DESIGN.md §5.2/§5.3 (truncated back substitution; complex LDL^T inverse of I - iK_oo:
    # LDL^T 4/3 o^3 with 4-product complex updates, L^-1 and Z^T D^-1 Z o^3 each with 3M), the
    # SURVEY §8(d) counts
    # beside them, FP64 DMMA fraction, and HBM GB/s from the committed ncu capture's bytes per launch
    fk_x, ft_x = 0.0, 0.0
    for s in range(args.warmup, nsteps):
        no = step_inputs[s]["no_host"].astype(np.float64)
        fk_x += float(np.sum((2.0 / 3.0) * nch ** 3 + nch ** 2 * no + no ** 3))
        ft_x += float(np.sum((10.0 / 3.0) * no ** 3))
    la = {}
    for kname, key, fx, fs in (("match_kernel", "match", fk_x, fk), ("tepi_kernel", "tepi", ft_x, ft)):
        ms_k, n_k = stats.get(key, (0.0, 0))
        if ms_k <= 0:
            continue
        tb, tsrc = ncu_traffic(args.config, batch, kernel=kname)
        # DRAM rate of the one launch ncu captured (its bytes over its own duration): the captured
        # block's n_open differs from this run's mix, so its bytes are not divided by this run's time
        tms = getattr(ncu_traffic, "duration_ms", 0.0) if tb else 0.0
        la[key] = {"ms": round(ms_k, 3), "launches": n_k,
                   "tflops_executed": fx / (ms_k / 1e3) / 1e12, "tflops_survey_count": fs / (ms_k / 1e3) / 1e12,
                   "frac_fp64_dmma_peak": fx / (ms_k / 1e3) / 1e12 / FP64_DMMA_PEAK_TFLOPS,
                   "ncu_dram_bytes_per_launch": tb,
                   "ncu_hbm_gbs": (tb / (tms / 1e3) / 1e9) if tb and tms else None,
                   "ncu_hbm_frac": (tb / (tms / 1e3) / 1e9 / float(measured_peaks().get("hbm_gbs", 6543.7)))
                   if tb and tms else None,
                   "traffic_source": tsrc}
    path_tflops = (fr + fk + ft) / (ms / 1e3) / 1e12
    ms_g, n_g = stats.get("i8gemm", (0.0, 0))

    # ---- the gathered result is complete and consistent on every rank -------------------------
    gather = None
    if world > 1:
        mine = torch.cat([o["rowsum"] for o in outs])
        idx = torch.from_numpy(shards[rank]).to(dev)
        assert torch.equal(full[idx], mine)
        covered = np.concatenate(shards)
        gather = {"energies": int(len(covered)), "bytes": int(len(covered) * nch * 8),
                  "inside_timed_region": True, "w_broadcast_s": round(bcast_s, 3),
                  "w_broadcast_bytes": int(w_d.numel() * 8)}

    # ---- end-to-end through the C ABI with host buffers ---------------------------------------
    e2e = None
    if not args.no_e2e:
        w_h = rmx.pinned_empty((nch, ldw))
        w_h[:] = w_d.cpu().numpy()
        Ek_h = rmx.pinned_empty((nlev,))
        Ek_h[:] = Ek_d.cpu().numpy()
        host_steps = []
        for s in range(nsteps):
            d = step_inputs[s]
            hs = {}
            for k in ("E", "F", "G", "Fp", "Gp"):
                buf = rmx.pinned_empty(tuple(d[k].shape))
                buf[:] = d[k].cpu().numpy()
                hs[k] = buf
            buf = rmx.pinned_empty(tuple(d["no"].shape), np.int32)
            buf[:] = d["no_host"]
            hs["no"] = buf
            hs["rowsum"] = rmx.pinned_empty((d["hi"] - d["lo"], nch))
            hs["status"] = rmx.pinned_empty((d["hi"] - d["lo"],), np.int32)
            host_steps.append(hs)

        def host_step(s):
            h = host_steps[s]
            return ctx.sweep_host(w_h, Ek_h, a, h["E"], h["F"], h["G"], h["Fp"], h["Gp"], h["no"],
                                  batch=batch, rowsum=h["rowsum"], status=h["status"])

        for s in range(args.warmup):
            host_step(s)
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        h2d = d2h = 0
        e0.record(stream)
        t0 = time.perf_counter()
        for s in range(args.warmup, nsteps):
            _, _, hb, db = host_step(s)
            h2d += hb
            d2h += db
        e1.record(stream)
        torch.cuda.synchronize()
        e_ms = max(e0.elapsed_time(e1), 1e3 * (time.perf_counter() - t0))
        if world > 1:
            t = torch.tensor([e_ms], dtype=torch.float64, device=dev)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            e_ms = float(t[0])
        e2e = {"value": n_energies / (e_ms / 1e3), "unit": "energies/s",
               "h2d_bytes_per_step": int(h2d // args.steps), "d2h_bytes_per_step": int(d2h // args.steps),
               "includes": "W, E_k, E, F, G, F', G', n_open H2D + rowsum, status D2H every step"}

    # ---- CPU oracle baseline (rank 0, N = 1 only) --------------------------------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        # (world == 1: rank 0 holds the generated case)
        sample = [case.ne // 2 + s for s in range(max(1, args.oracle_sample))]
        if args.config in ("tiny", "small"):
            sample = list(range(0, case.ne, max(1, case.ne // 256)))
        threads = os.cpu_count() or 1
        v, dt = oracle_baseline(case, sample, threads)
        cpu = {"value": v, "unit": "energies/s", "cores": threads, "kind": "oracle",
               "sample": f"{len(sample)} energies of {args.config} (mesh index {sample[0]}..{sample[-1]}), "
                         f"{dt:.1f} s, OpenMP over rows/energies"}

    if rank == 0:
        if args.r_algo == "int8" and ms_g > 0:  # (nch < 256 falls back to the DMMA R formation)
            # dominant kernel: the INT8 tensor-core GEMMs of the CRT R formation. Algorithmic int8 ops per
            # energy: 16 moduli x nch(nch+1) nlev (upper triangle, like the fp64 count). Peak: the INT8 dense
            # rate = measured bf16 (sustained: the GEMMs run inside a long step) x the nominal int8/bf16 ratio 2.
            pk = measured_peaks()
            peak_i8 = 2.0 * float(pk.get("bf16_tflops_sustained", 1378.4))
            ops_i8 = 16.0 * fr
            ach_i8 = ops_i8 / (ms_g / 1e3) / 1e12 if ms_g > 0 else None
            # DRAM bytes per GEMM launch (one chunk of 8 energies: librmx kInt8Chunk)
            traffic, traffic_src = ncu_traffic(args.config, min(batch, 8), kernel="oz_gemm")
            roofline = {"bound": "tensor", "kernel": "oz_gemm2_kernel (INT8 tcgen05 cta_group::2, 256x256 upper-triangle blocks, 16 moduli, CRT R formation)",
                        "achieved": ach_i8, "peak": peak_i8, "unit": "TOPS",
                        "frac": (ach_i8 / peak_i8) if ach_i8 else None,
                        "traffic": traffic, "traffic_source": traffic_src,
                        "peak_source": "2 x bf16_tflops_sustained of MEASURED_PEAKS.json (nominal int8/bf16 ratio, "
                                       "B200_PROFILING.md); nominal dense int8 4500 TOPS",
                        "algorithmic": "16 x nch(nch+1) x nlev int8 ops per energy x energies per launch",
                        "traffic_per": "one oz_gemm2 launch = 8 energies (algorithmic bytes: 8 x 16 x nch x nlev "
                                       "X residues + 16 x nch x nlev W residues)"}
            r_form = {"algo": "int8-crt (rint8.cu)", "fp64_equivalent_tflops": achieved_r,
                      "vs_fp64_dmma_peak": (achieved_r / FP64_DMMA_PEAK_TFLOPS) if achieved_r else None,
                      "i8gemm_ms": round(ms_g, 3), "rform_total_ms": round(ms_r, 3)}
        else:
            traffic, traffic_src = ncu_traffic(args.config, batch)
            roofline = {"bound": "tensor", "kernel": "rform (FP64 DMMA R formation)",
                        "achieved": achieved_r, "peak": FP64_DMMA_PEAK_TFLOPS, "unit": "TFLOP/s",
                        "frac": (achieved_r / FP64_DMMA_PEAK_TFLOPS) if achieved_r else None,
                        "traffic": traffic, "traffic_source": traffic_src,
                        "peak_source": "measured FP64 DMMA.8x8x4 peak, tools/fp64_peak.cu on this pool "
                                       "(profiles/r01_fp64_peak.jsonl); MEASURED_PEAKS.json has no FP64 entry",
                        "algorithmic": "nch(nch+1)*nlev flops per energy x energies per launch"}
            r_form = {"algo": "fp64-dmma (rform.cu)"}
        line = {
            "metric": "energies/sec (R->K->|T|^2 sweep)",
            "value": value, "unit": "energies/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None,
            "dtype": "f64" if r_form["algo"].startswith("fp64") else "f64 (R: exact int8 CRT on tcgen05; K, T: f64 DMMA)",
            "data": "synthetic (rmx_synth, seed 0)",
            "config": {"workload": args.config, "nch": nch, "nlev": nlev, "ne_mesh": ne,
                       "a": cfg["a"], "energies_per_step_per_gpu": batch,
                       "parallelism": f"energy-sharded block-cyclic x{world}",
                       "l2": f"inputs exceed L2 (W = {nch * nlev * 8 / 1e6:.0f} MB, 126 MB L2)"
                       if nch * nlev * 8 > 126e6 else "W fits L2; R/K batch buffers exceed L2"},
            "roofline": roofline,
            "r_formation": r_form,
            "kernel_ms": {k: round(v[0], 3) for k, v in stats.items() if k != "launches"},
            "la_kernels": la,
            "path_fp64_tflops": path_tflops,
            ("path_fp64_frac" if r_form["algo"].startswith("fp64") else "path_fp64_equivalent_vs_dmma_peak"):
                path_tflops / FP64_DMMA_PEAK_TFLOPS,
            "gpu_launches": int(stats["launches"]),
            "bad_status_energies": bad,
            "clocks": clk.summary(),
            "e2e": e2e,
            "cpu_baseline": cpu,
            "setup_s": round(setup_s, 2),
            "gather": gather,
            "timing": {"runs_ms": [round(x, 3) for x in runs_ms], "value_from": f"median of {args.repeats} "
                       "uninstrumented runs of K steps", "instrumented_run_ms": round(ms_instr, 3),
                       "kernel_breakdown_from": "a separate run with per-launch CUDA events (kernel_ms, "
                       "roofline.achieved, la_kernels)"},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
