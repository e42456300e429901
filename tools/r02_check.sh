#!/usr/bin/env bash
# Quick HEAD check: GPU suite, smoke, C2 line, C3 line
OUT=gpurun_out/${1:-check}
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $OUT/gpu.txt
timeout 2400 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.txt 2>&1; tail -3 $OUT/pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1; tail -1 $OUT/smoke.txt
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; tail -c 300 $OUT/bench.json
timeout 600 python bench.py --config c3 --no-cpu-baseline > $OUT/c3.json 2>$OUT/c3.err; tail -c 300 $OUT/c3.json
