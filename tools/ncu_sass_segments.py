"""Summarise an ncu --page source (SASS) CSV: warp-stall samples per function segment (split at
RET/EXIT) and the top instructions. Usage: ncu -i X.ncu-rep --page source --csv --print-source sass > f.csv;
python tools/ncu_sass_segments.py f.csv"""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[hdr_i]
col = {h: i for i, h in enumerate(hdr)}
data = [r for r in rows[hdr_i + 1:] if len(r) == len(hdr)]
S = col["Warp Stall Sampling (All Samples)"]
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(int(r[S]) for r in data)
print("total samples", tot)
seg, segs = [], []
for r in data:
    seg.append(r)
    if "RET" in r[1] or "EXIT" in r[1]:
        segs.append(seg); seg = []
if seg: segs.append(seg)
for k, s in enumerate(segs):
    n = sum(int(r[S]) for r in s)
    if n < 0.005 * tot: continue
    st = collections.Counter()
    for r in s:
        for h in stall_cols:
            st[h] += int(r[col[h]] or 0)
    calls = [r[1].strip() for r in s if "CALL" in r[1]][:6]
    top = sorted(s, key=lambda r: -int(r[S]))[:6]
    print(f"\n== segment {k}: {len(s)} instrs, {n} samples ({100*n/tot:.1f}%) first: {s[0][1].strip()}")
    print("   stalls:", ", ".join(f"{h[6:]}={100*v/n:.0f}%" for h, v in st.most_common(5)))
    if calls: print("   calls:", calls)
    for r in top:
        print(f"   {int(r[S]):7d}  {r[1].strip()[:90]}")
