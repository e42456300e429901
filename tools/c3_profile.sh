#!/usr/bin/env bash
OUT=gpurun_out/${1:-c3prof}
mkdir -p $OUT
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 2000 -c 600 --csv \
  --log-file $OUT/launches.csv python bench.py --config c3 --steps 1 --warmup 3 > $OUT/run.log 2>&1
echo "ncu rc $?"
python tools/launch_summary.py $OUT/launches.csv $OUT/launches_summary.txt > /dev/null 2>&1
cat $OUT/launches_summary.txt
