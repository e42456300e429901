# SPDX-License-Identifier: Apache-2.0
"""Summarise an `ncu --metrics gpu__time_duration.sum` launch list (csv) per kernel."""
import collections
import csv
import sys


def main(src, dst):
    rows = list(csv.reader(open(src)))
    start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[start]
    ki, mv, mu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    agg = collections.OrderedDict()
    for r in rows[start + 1:]:
        if len(r) <= mv:
            continue
        v = float(r[mv].replace(",", "")) * scale.get(r[mu], 1.0)
        a = agg.setdefault(r[ki][:64], [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(a[1] for a in agg.values())
    lines = ["kernel                                                            launches  total_us  share"
             "  (ncu, serialised; compare shares, not absolute times)"]
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"{k:64s} {n:6d} {t:10.1f}  {t / tot:.3f}")
    open(dst, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main(*sys.argv[1:3])
