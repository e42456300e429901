timeout 900 python -m pytest tests/test_engine_gpu.py tests/test_gemm_gpu.py -x -q > gpurun_out/ext_engine.log 2>&1; tail -3 gpurun_out/ext_engine.log
AB_VARIANTS=nofold bash tools/r02_ab2.sh
