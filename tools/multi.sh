#!/usr/bin/env bash
# torchrun logic check on one GPU (ranks share the device) + the other configs' bench lines
OUT=gpurun_out/${1:-multi}
mkdir -p $OUT
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline > $OUT/tr2.txt 2>&1
echo "torchrun ours rc $?"; tail -1 $OUT/tr2.txt | cut -c1-400
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29534 bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > $OUT/tr2ref.txt 2>&1
echo "torchrun reference rc $?"; tail -1 $OUT/tr2ref.txt | cut -c1-300
bash tools/configs.sh ${1:-multi}/configs
