#!/usr/bin/env bash
# memcheck / synccheck over this round's later paths: streamed PLT1 ingest (chunk scatter
# kernel), bulk registration, peer migration, decode graph replay + split FFN2 + wide head.
OUT=gpurun_out/${1:-sanitize_new}
mkdir -p $OUT
for tool in memcheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python -m pytest -x -q -m gpu \
    tests/test_ingest.py::test_gpu_streamed_plt1_format_errors tests/test_ingest.py::test_gpu_bulk_registration \
    tests/test_rebalance.py::test_migrate_and_replicate_same_process \
    "tests/test_engine_gpu.py::test_generate_graph_replay_matches_eager" > $OUT/new_$tool.txt 2>&1
  echo "new paths $tool rc $? :: $(grep -E 'ERROR SUMMARY|passed|failed' $OUT/new_$tool.txt | head -4 | tr '\n' ' ')"
done
