"""Per-CUDA-source-line warp-stall samples of one kernel in an ncu report:
   python tools/ncu_lines.py REPORT.ncu-rep KERNEL_REGEX [N]"""
import csv, collections, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "-k", f"regex:{kern}", "--page", "source", "--csv",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
cur, hdr, agg, src = None, None, collections.Counter(), {}
stalls = collections.defaultdict(collections.Counter)
for r in rows:
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 6:
        continue
    try:
        ln = int(r[0])
        v = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
    except ValueError:
        continue
    agg[(cur, ln)] += v
    src[(cur, ln)] = r[1]
    for h, x in zip(hdr, r):
        if h.startswith("stall_") and "Not Issued" not in h:
            try:
                stalls[(cur, ln)][h[6:]] += int(x)
            except ValueError:
                pass
tot = sum(agg.values()) or 1
print("total samples", tot)
for (f, ln), v in agg.most_common(top):
    st = ", ".join(f"{k}={100 * x / max(v, 1):.0f}%" for k, x in stalls[(f, ln)].most_common(3))
    print(f"{100 * v / tot:5.1f}% {f}:{ln} {src[(f, ln)].strip()[:70]}   [{st}]")
