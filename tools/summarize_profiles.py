"""Summarise a round's ncu artefacts into profiles/:
  python tools/summarize_profiles.py ROUND [launches.csv] [report.ncu-rep]
writes profiles/rROUND_launches.md (per-kernel share of the launch list) and
profiles/rROUND_ncu_kernels.json (per-kernel key metrics of the full capture; bench.py reads the
R-formation DRAM traffic from it for roofline.traffic)."""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rnd = sys.argv[1] if len(sys.argv) > 1 else "01"
launches = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "gpurun_out", "launches.csv")
rep = sys.argv[3] if len(sys.argv) > 3 else os.path.join(ROOT, "gpurun_out", "prof_round.ncu-rep")
out_dir = os.path.join(ROOT, "profiles")

# ---- launch list ("-" skips it) ----------------------------------------------------------------
rows = list(csv.reader(open(launches))) if launches != "-" else []
hi = next((i for i, r in enumerate(rows) if r and r[0] == "ID"), None)
hdr = rows[hi] if hi is not None else []
col = {h: i for i, h in enumerate(hdr)}
agg = collections.OrderedDict()
scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3, "ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}
for r in (rows[hi + 1:] if hi is not None else []):
    if len(r) != len(hdr) or r[col["Metric Name"]] != "gpu__time_duration.sum":
        continue
    name = r[col["Kernel Name"]].split("(")[0][:70]
    v = float(r[col["Metric Value"]].replace(",", "")) * scale[r[col["Metric Unit"]]]
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += v
tot = sum(v[1] for v in agg.values()) or 1.0
ours = {k: v for k, v in agg.items() if any(s in k for s in ("rform", "match_kernel", "tepi_kernel", "oz_",
                                                                "dipole_g", "conv_gauss", "maxwell"))}
tot_ours = sum(v[1] for v in ours.values()) or 1.0
lines = [f"# Round {rnd} ncu launch list (gpu__time_duration.sum, --clock-control none)", "",
         "Command: `python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --repeats 1` (darc, 296 energies/step, "
         "INT8-CRT R formation).",
         "Per-launch times are cold-cache and serialised: compare shares, not absolutes.", "",
         "| kernel | launches | total ms | share of all | share of librmx |", "|---|---|---|---|---|"]
for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:15]:
    lines.append(f"| `{k}` | {v[0]} | {v[1]:.1f} | {100 * v[1] / tot:.1f}% | "
                 f"{(100 * v[1] / tot_ours) if k in ours else 0:.1f}% |")
if agg:
    open(os.path.join(out_dir, f"r{rnd}_launches.md"), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))

# ---- full capture ------------------------------------------------------------------------------
metrics = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
           "lts__t_sector_hit_rate.pct", "launch__registers_per_thread", "launch__grid_size",
           "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
           "smsp__inst_executed.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed"]
if os.path.exists(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    h = rr[0]
    units = dict(zip(h, rr[1]))
    res = {}
    for r in rr[2:]:
        d = dict(zip(h, r))
        name = d["Kernel Name"].split("(")[0]
        ent = {}
        for m in metrics:
            v = d.get(m)
            try:
                ent[m] = float(v.replace(",", ""))
            except (AttributeError, ValueError):
                ent[m] = None
            ent[m + ".unit"] = units.get(m)
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            f = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(units.get(m), None)
            if f and ent[m] is not None and ent[m] == ent[m]:
                ent[m.replace(".sum", ".bytes")] = ent[m] * f
        if "oz_" in name:  # INT8-CRT kernels: one launch = one chunk of 8 energies (kInt8Chunk at darc)
            ent["workload"] = {"config": "darc", "energies_per_launch": 8,
                               "note": "one launch = one chunk of 8 energies (x 16 moduli)"}
        else:
            ent["workload"] = {"config": "darc", "energies_per_launch": 296}
        res.setdefault(name, ent)
    path = os.path.join(out_dir, f"r{rnd}_ncu_kernels.json")
    old = json.load(open(path)) if os.path.exists(path) else {}
    old.update(res)  # kernels captured in this report replace their older entries
    json.dump(old, open(path, "w"), indent=1)
    for k, v in res.items():
        print(k, {m: v[m] for m in metrics[:5]})
