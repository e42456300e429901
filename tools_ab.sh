#!/usr/bin/env bash
# Same-box A/B of engine variants (env var settings) on quick timed-region runs.
#   bash tools_ab.sh OUTDIR "VAR=a" "VAR=b" ...
OUT=gpurun_out/${1:-ab}
shift
mkdir -p $OUT
for rep in 1 2; do
  for v in "$@"; do
    tag=$(echo "$v" | tr '= ' '__')
    env $v timeout 600 python bench.py --no-cpu-baseline --steps 40 > $OUT/$tag.$rep.json 2>&1
    python3 - "$OUT/$tag.$rep.json" "$v rep$rep" <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
k = {n: round(v["ms_per_launch"] * 1e3, 1) for n, v in d["kernels"].items()}
print(sys.argv[2], round(d["value"]), round(d["ms_per_step"], 3), d.get("clocks", {}).get("sm_mhz"), k)
PY
  done
done
