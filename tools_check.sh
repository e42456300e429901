#!/usr/bin/env bash
# Box check: GPU tests, C4 swap A/B (batched vs per-copy H2D), 2-rank torchrun logic.
mkdir -p gpurun_out/check
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/check/pytest.txt 2>&1; echo "pytest rc $?"
tail -3 gpurun_out/check/pytest.txt
for v in HMI_BATCH_COPY=0 HMI_BATCH_COPY=1 HMI_BATCH_COPY=0 HMI_BATCH_COPY=1; do
  env $v timeout 600 python bench.py --config c4 --quick --no-cpu-baseline > gpurun_out/check/c4_$v.json 2>&1
  echo "$v $(tail -1 gpurun_out/check/c4_$v.json | cut -c1-400)"
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/check/tr2.txt 2>&1
echo "torchrun rc $?"; tail -2 gpurun_out/check/tr2.txt | cut -c1-600
