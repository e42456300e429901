timeout 900 python -m pytest -q tests/test_shard_gpu.py tests/test_cpp_backend.py "tests/test_engine_gpu.py::test_token_tag_head" > gpurun_out/t3.log 2>&1; tail -5 gpurun_out/t3.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/b3_c2.json 2>gpurun_out/b3_c2.err; tail -c 600 gpurun_out/b3_c2.json
timeout 900 python bench.py --config c4 --pool-fraction 0.5 --no-cpu-baseline > gpurun_out/b3_c4_05.json 2>gpurun_out/b3_c4.err; tail -c 1200 gpurun_out/b3_c4_05.json
timeout 900 python bench.py --config c4 --pool-fraction 1.0 --no-cpu-baseline > gpurun_out/b3_c4_10.json 2>>gpurun_out/b3_c4.err; tail -c 300 gpurun_out/b3_c4_10.json
tail -5 gpurun_out/b3_c4.err
