#!/usr/bin/env bash
# compute-sanitizer over the smoke batch (all four tools) and the swap / decode paths
# (memcheck, synccheck); every report is then classified by tools/sanitize_classify.py
OUT=gpurun_out/${1:-sanitize_r02}
mkdir -p $OUT
for tool in memcheck synccheck racecheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 100000 \
    python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$tool.txt 2>&1
  echo "smoke $tool rc $?"
done
for tool in memcheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 200 python -m pytest -x -q -m gpu \
    tests/test_engine_gpu.py -k "swap or s256 or s512 or generate_graph or wide_bottleneck" > $OUT/paths_$tool.txt 2>&1
  echo "paths $tool rc $? :: $(grep -E 'ERROR SUMMARY|passed|failed' $OUT/paths_$tool.txt | head -4 | tr '\n' ' ')"
done
