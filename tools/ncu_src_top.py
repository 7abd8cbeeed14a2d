"""Top SASS lines of an `ncu --page source --csv` export by stall samples,
with their dominant stall reasons and shared-memory conflicts.

    python tools/ncu_src_top.py gpurun_out/q6_src.csv [--n 30]
"""
import argparse
import csv
from collections import Counter

ap = argparse.ArgumentParser()
ap.add_argument("csv")
ap.add_argument("--n", type=int, default=30)
a = ap.parse_args()
rows = list(csv.reader(open(a.csv)))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = Counter()
lines = []
for r in rows[2:]:
    if r and r[0] == "Kernel Name":
        break  # first kernel's block only
    if len(r) != len(hdr) or not r[ix["Warp Stall Sampling (All Samples)"]].isdigit():
        continue
    d = {h: r[ix[h]] for h in hdr}
    n = int(d["Warp Stall Sampling (All Samples)"] or 0)
    st = {s: int(d[s] or 0) for s in stalls}
    tot.update(st)
    lines.append((n, d["Address"][-5:], d["Source"].strip()[:60], st,
                  d.get("L1 Wavefronts Shared Excessive", ""), d.get("L1 Wavefronts Shared", "")))
all_n = sum(tot.values())
print("total samples", all_n)
for s, v in tot.most_common(10):
    print(f"  {s:24s} {v:8d} {100 * v / max(1, all_n):5.1f}%")
print()
for n, addr, src, st, ex, wf in sorted(lines, key=lambda x: -x[0])[:a.n]:
    top = ", ".join(f"{k[6:]}={v}" for k, v in Counter(st).most_common(2) if v)
    print(f"{n:7d} {addr} {src:60s} {top}  smem_wf={wf} excess={ex}")
