# SPDX-License-Identifier: Apache-2.0
"""Top SASS lines by warp-stall samples per kernel from `ncu --page source --csv --print-source sass`:
python tools/ncu_sass_hot.py source.csv [kernel-substring] [top]"""
import csv
import sys

path = sys.argv[1]
want = sys.argv[2] if len(sys.argv) > 2 else ""
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
rows, name, hdr = [], None, None
blocks = []
with open(path) as fh:
    for r in csv.reader(fh):
        if r and r[0] == "Kernel Name":
            if name is not None:
                blocks.append((name, hdr, rows))
            name, hdr, rows = r[1], None, []
        elif r and r[0] == "Address":
            hdr = r
        elif hdr is not None and r:
            rows.append(r)
if name is not None:
    blocks.append((name, hdr, rows))
seen = set()
for name, hdr, rows in blocks:
    if want not in name or (name in seen):
        continue
    seen.add(name)
    iS = hdr.index("Warp Stall Sampling (All Samples)")
    stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    tot = sum(float(r[iS] or 0) for r in rows)
    print(f"=== {name}  samples {tot:.0f}")
    agg = {}
    for r in rows:
        for i in stall_cols:
            agg[hdr[i]] = agg.get(hdr[i], 0) + float(r[i] or 0)
    print("   ", ", ".join(f"{k[6:]} {v / max(tot, 1):.0%}" for k, v in sorted(agg.items(), key=lambda x: -x[1])[:8]))
    for r in sorted(rows, key=lambda r: -float(r[iS] or 0))[:top]:
        st = sorted(((hdr[i][6:], float(r[i] or 0)) for i in stall_cols), key=lambda x: -x[1])[:2]
        print(f"  {float(r[iS] or 0) / max(tot, 1):6.1%} {r[0]:>6} {r[1][:70]:70s} {st}")
