# ncu --set full of one layer's attention, grouped down GEMM and the step's retrieval
OUT=gpurun_out/ncu_at
mkdir -p $OUT
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"attention_tc|retrieve|gemm_tcgen05_kernel" -s 30 -c 4 \
  -o $OUT/prof python bench.py --quick --steps 2 --warmup 3 --no-cpu-baseline > $OUT/ncu_run.log 2>&1
echo "ncu rc $?"; tail -2 $OUT/ncu_run.log
ncu -i $OUT/prof.ncu-rep --page details --csv > $OUT/details.csv 2>/dev/null
ncu -i $OUT/prof.ncu-rep --page source --csv --print-source sass > $OUT/source.csv 2>/dev/null
python tools/ncu_details.py $OUT/details.csv > $OUT/details.txt 2>/dev/null
