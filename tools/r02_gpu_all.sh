# Round-2 GPU pass: all -m gpu tests (including the at-scale parity suite), results in gpurun_out/
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
lscpu > gpurun_out/lscpu.txt
HMI_PARITY_OUT=gpurun_out/parity timeout 3000 python -m pytest tests -m gpu -q --durations=40 ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1
tail -70 gpurun_out/pytest_gpu.log
