#!/usr/bin/env bash
# A/B the LayerNorm placements on one box (same clocks): quick timed-region runs.
OUT=gpurun_out/${1:-ab}
mkdir -p $OUT
for rep in 1 2; do
  for m in fold unfused; do
    HMI_LN_MODE=$m timeout 600 python bench.py --no-cpu-baseline --quick --steps 40 > $OUT/$m.$rep.json 2>&1
    echo "$m rep$rep $(tail -1 $OUT/$m.$rep.json)"
  done
done
