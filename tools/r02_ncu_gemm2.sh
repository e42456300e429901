# ncu --set full of one layer's four pair-kernel GEMMs (QKV, O+ext, FFN1, FFN2) + the grouped down GEMM
OUT=gpurun_out/ncu_g2
mkdir -p $OUT
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"gemm" -s 50 -c 5 \
  -o $OUT/prof python bench.py --quick --steps 2 --warmup 3 --no-cpu-baseline > $OUT/ncu_run.log 2>&1
echo "ncu rc $?"; tail -3 $OUT/ncu_run.log
ncu -i $OUT/prof.ncu-rep --page details --csv > $OUT/details.csv 2>/dev/null
ncu -i $OUT/prof.ncu-rep --page raw --csv > $OUT/raw.csv 2>/dev/null
ncu -i $OUT/prof.ncu-rep --page source --csv --print-source sass > $OUT/source.csv 2>/dev/null
python tools/ncu_details.py $OUT/details.csv > $OUT/details.txt 2>/dev/null
ls -la $OUT
