# SPDX-License-Identifier: Apache-2.0
"""SASS window with stall samples: python tools/ncu_window.py source.csv kernel-substr lo hi [lo hi ...]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = []
        blocks.append((r[1], cur))
    elif r and r[0].startswith("0x") and cur is not None:
        cur.append(r)
name, ins = [b for b in blocks if sys.argv[2] in b[0]][0]
a = sys.argv[3:]
for lo, hi in zip(a[::2], a[1::2]):
    print("---")
    for i in range(int(lo), int(hi)):
        print(i, ins[i][2], ins[i][1][:100])
