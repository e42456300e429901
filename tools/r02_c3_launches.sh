#!/usr/bin/env bash
# GPU suite, the C3 line, and the ncu launch list of C3 decode steps (serialised per-kernel
# durations; the shares, not the absolute times, compare with the bench's profile pass)
OUT=gpurun_out/${1:-c3l}
mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.txt 2>&1; tail -2 $OUT/pytest_gpu.txt
timeout 600 python bench.py --config c3 --no-cpu-baseline > $OUT/c3.json 2>$OUT/c3.err; tail -c 200 $OUT/c3.json; echo
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 600 --csv \
  --log-file $OUT/launches.csv python bench.py --config c3 --steps 1 --warmup 3 --no-cpu-baseline > $OUT/ncu_run.log 2>&1
echo "ncu rc $?"
python tools/launch_summary.py $OUT/launches.csv $OUT/launches_summary.txt > /dev/null 2>&1; cat $OUT/launches_summary.txt
