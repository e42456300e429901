#!/usr/bin/env bash
# ncu --set full of decode-step K-split GEMMs (gemm_dec_kernel) in the C3 config
OUT=gpurun_out/${1:-ncudec}
mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_dec -s ${2:-40} -c ${3:-8} \
  -o $OUT/prof python bench.py --config c3 --steps 1 --warmup 3 --no-cpu-baseline > $OUT/run.log 2>&1
echo "ncu rc $?"
ncu -i $OUT/prof.ncu-rep --page details --csv > $OUT/details.csv 2>/dev/null
python tools/ncu_details.py $OUT/details.csv > $OUT/details.txt; head -120 $OUT/details.txt
ncu -i $OUT/prof.ncu-rep --page raw --csv > $OUT/raw.csv 2>/dev/null
