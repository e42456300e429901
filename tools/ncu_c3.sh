#!/usr/bin/env bash
OUT=gpurun_out/${1:-ncuc3}
mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$2" -s 40 -c 1 \
  -o $OUT/prof python bench.py --config c3 --steps 1 --warmup 3 --no-cpu-baseline > $OUT/run.log 2>&1
echo "ncu rc $?"
ncu -i $OUT/prof.ncu-rep --page details --csv > $OUT/details.csv 2>/dev/null
ncu -i $OUT/prof.ncu-rep --page source --csv --print-source sass > $OUT/source.csv 2>/dev/null
python tools/ncu_details.py $OUT/details.csv
python tools/ncu_hot.py $OUT/source.csv "" 14
