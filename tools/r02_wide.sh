# 256 x 512 pair units for QKV / FFN1: kernel tests, then same-box A/B against the previous commit
timeout 600 python -m pytest tests/test_gemm_gpu.py -x -q -s -k "wide" > gpurun_out/wide_tests.log 2>&1; grep -E "wide|passed|failed" gpurun_out/wide_tests.log | tail -8
timeout 900 python -m pytest tests/test_engine_gpu.py tests/test_gemm_gpu.py -x -q > gpurun_out/wide_engine.log 2>&1; tail -2 gpurun_out/wide_engine.log
AB_VARIANTS=prev bash tools/r02_ab2.sh
AB_VARIANTS=prev bash tools/r02_ab2.sh
