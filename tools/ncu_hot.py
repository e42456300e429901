# SPDX-License-Identifier: Apache-2.0
"""Top stalled SASS instructions per kernel from `ncu --page source --csv --print-source sass`.
python tools/ncu_hot.py source.csv [kernel-substring] [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
want = sys.argv[2] if len(sys.argv) > 2 else ""
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "ins": []}
        blocks.append(cur)
    elif r and r[0].startswith("0x") and cur is not None:
        cur["ins"].append((int(r[2] or 0), r[1].strip(), r[0]))
seen = set()
for b in blocks:
    if want not in b["name"] or b["name"] in seen:
        continue
    seen.add(b["name"])
    tot = sum(s for s, _, _ in b["ins"]) or 1
    print(f"=== {b['name'][:90]}  total samples {tot}")
    idx = {a: i for i, (_, _, a) in enumerate(b["ins"])}
    for s, src, a in sorted(b["ins"], reverse=True)[:top]:
        print(f"  {100.0 * s / tot:5.1f}%  [{idx[a]:5d}] {src[:100]}")
