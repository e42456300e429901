#!/usr/bin/env bash
# in-step GEMM metrics of the current tree vs an older build (build/ab/<x>)
M=gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second,launch__grid_size
for tree in . "$@"; do
  echo "== $tree"
  (cd $tree && timeout 600 ncu --metrics $M --clock-control none -k regex:"gemm2|adapter" -s 60 -c 10 --csv \
     python bench.py --quick --steps 2 --warmup 3 --no-cpu-baseline 2>/dev/null) > /tmp/ab.csv
  python3 - /tmp/ab.csv <<'PY'
import csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]; ix = {h: i for i, h in enumerate(hdr)}
cur = {}
for r in rows[1:]:
    key = (r[ix["ID"]], r[ix["Kernel Name"]][:34])
    cur.setdefault(key, {})[r[ix["Metric Name"]]] = r[ix["Metric Value"]]
for (i, k), m in cur.items():
    print(i, k, {n.split("__")[1][:18]: v for n, v in m.items()})
PY
done
