#!/usr/bin/env bash
# Run-to-run spread of the headline on one box: default steps, longer timed regions, and
# without the nvidia-smi clock sampler.
v() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', round(d['value']), round(d['e2e']['value']), round(d['ms_per_step'],3))"; }
for rep in 1 2 3; do
  timeout 600 python bench.py --no-cpu-baseline 2>/dev/null | v "steps20"
  timeout 600 python bench.py --no-cpu-baseline --steps 100 2>/dev/null | v "steps100"
  HMI_BENCH_NO_CLOCKS=1 timeout 600 python bench.py --no-cpu-baseline 2>/dev/null | v "steps20_noclk"
done
