#!/usr/bin/env bash
# same-box A/B of the C3 (hGPT-2 small generation) bench line: current tree vs build/ab/<tree>
for rep in 1 2; do
  for tree in . "$@"; do
    (cd $tree && timeout 900 python bench.py --config c3 --no-cpu-baseline --steps 5 --warmup 3 2>/dev/null) | python3 -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$tree', round(d['value']), round(d['ms_per_step'],2), {k: round(v['ms_per_launch']*1e3,1) for k,v in d.get('kernels',{}).items()})"
  done
done
