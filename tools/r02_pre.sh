timeout 900 python -m pytest tests/test_engine_gpu.py tests/test_gemm_gpu.py -x -q > gpurun_out/pre_tests.log 2>&1; tail -2 gpurun_out/pre_tests.log
AB_VARIANTS=prev bash tools/r02_ab2.sh
AB_VARIANTS=prev bash tools/r02_ab2.sh
