#!/usr/bin/env bash
# C4 (10k tenants, adapters swapped from pinned host memory): HBM slot pool sweep
OUT=gpurun_out/${1:-c4sweep}
mkdir -p $OUT
for f in 0.5 0.7 0.8 0.9 1.0; do
  timeout 900 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline --pool-fraction $f > $OUT/c4_$f.json 2> $OUT/c4_$f.err
  python3 - $OUT/c4_$f.json $f <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
k = d["kernels"]
comp = sum(v["ms_per_launch"] * v["launches"] for n, v in k.items()) / d["steps"]
print(f"pool {sys.argv[2]}: {d['value']:.0f} req/s, step {d['ms_per_step']:.3f} ms, kernels {comp:.3f} ms/step, "
      f"e2e {d['e2e']['value']:.0f} req/s, copied {d['pool']['bytes_copied'] / 1e9:.2f} GB total")
PY
done
