# ncu of consecutive decode-step GEMMs of the C3 config (after the prefill's launches)
OUT=gpurun_out/${1:-ncuc3g}
mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tcgen05 -s ${2:-80} -c ${3:-10} \
  -o $OUT/prof python bench.py --config c3 --steps 1 --warmup 3 --no-cpu-baseline > $OUT/run.log 2>&1
echo "ncu rc $?"
ncu -i $OUT/prof.ncu-rep --page details --csv > $OUT/details.csv 2>/dev/null
python tools/ncu_details.py $OUT/details.csv
