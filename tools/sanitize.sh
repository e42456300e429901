#!/usr/bin/env bash
# compute-sanitizer over the smoke batch and the GEMM / adapter kernels (memcheck, racecheck,
# synccheck, initcheck); summaries into gpurun_out/<out>/
OUT=gpurun_out/${1:-sanitize}
mkdir -p $OUT
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 \
    python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$tool.txt 2>&1
  echo "smoke $tool rc $? :: $(grep -E 'ERROR SUMMARY|smoke ok|Error' $OUT/smoke_$tool.txt | head -3 | tr '\n' ' ')"
done
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gemm_gpu.py -x -q \
  -k "cta_pair or grouped or wave_tail" > $OUT/gemm_memcheck.txt 2>&1
echo "gemm memcheck rc $? :: $(grep -E 'ERROR SUMMARY|passed|failed' $OUT/gemm_memcheck.txt | head -3 | tr '\n' ' ')"
