#!/usr/bin/env bash
# ncu --set full of selected kernels inside the C2 step:  bash tools/ncu_kernel.sh OUT REGEX COUNT [skip]
OUT=gpurun_out/${1:-ncuk}
mkdir -p $OUT
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"$2" -s ${4:-20} -c ${3:-2} \
  -o $OUT/prof python bench.py --quick --steps 2 --warmup 3 --no-cpu-baseline > $OUT/ncu_run.log 2>&1
echo "ncu rc $?"; tail -3 $OUT/ncu_run.log
ncu -i $OUT/prof.ncu-rep --page details --csv > $OUT/details.csv 2>/dev/null
ncu -i $OUT/prof.ncu-rep --page source --csv --print-source sass > $OUT/source.csv 2>/dev/null
ls -la $OUT
