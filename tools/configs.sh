#!/usr/bin/env bash
# One line per BASELINE config on one GPU: C1, C3 (generation), C4 (10k tenants, 60% pool), C5 (hBERT-large)
OUT=gpurun_out/${1:-configs}
mkdir -p $OUT
for c in c1 c4 c5 c3; do
  timeout 1200 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > $OUT/$c.json 2> $OUT/$c.err
  echo "$c rc $? $(tail -1 $OUT/$c.json | cut -c1-700)"
  tail -2 $OUT/$c.err
done
