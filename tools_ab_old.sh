#!/usr/bin/env bash
# same-box A/B of the current tree against older builds copied to build/ab/<commit>
for rep in 1 2; do
  for tree in . "$@"; do
    (cd $tree && timeout 600 python bench.py --no-cpu-baseline --steps 20 2>/dev/null) | python3 -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$tree', round(d['value']), {k: round(v['ms_per_launch']*1e3,1) for k,v in d['kernels'].items()})"
  done
done
