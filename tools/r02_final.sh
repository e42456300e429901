#!/usr/bin/env bash
# Round-2 evidence pass at HEAD: GPU suite (+ parity records), smoke, C2 line (fp16 and bf16),
# every other config, the reference arm, the C2 ncu launch list and one ncu --set full layer
OUT=gpurun_out/${1:-r02end}
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $OUT/gpu.txt
HMI_PARITY_OUT=$OUT/parity timeout 2400 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.txt 2>&1; tail -2 $OUT/pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1; tail -1 $OUT/smoke.txt
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; tail -c 400 $OUT/bench.json
timeout 900 python bench.py --precision 1 --no-cpu-baseline > $OUT/bench_bf16.json 2> $OUT/bench_bf16.err
for c in c1 c3 c5 plot; do
  timeout 1200 python bench.py --config $c --no-cpu-baseline > $OUT/$c.json 2> $OUT/$c.err
  echo "$c rc $? $(tail -1 $OUT/$c.json | cut -c1-200)"
done
for p in 1.0 0.5; do
  timeout 1200 python bench.py --config c4 --pool-fraction $p --no-cpu-baseline --steps 60 > $OUT/c4_$p.json 2> $OUT/c4_$p.err
  echo "c4 $p rc $? $(tail -1 $OUT/c4_$p.json | cut -c1-200)"
done
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/ref.json 2> $OUT/ref.err; tail -c 300 $OUT/ref.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemm|attention|retrieve|route|fetch|head|scatter" -s 400 -c 120 --csv \
  --log-file $OUT/launches.csv python bench.py --quick --steps 3 --warmup 3 --no-cpu-baseline > $OUT/ncu_launch_run.log 2>&1
python tools/launch_summary.py $OUT/launches.csv $OUT/launches_summary.txt > /dev/null 2>&1; cat $OUT/launches_summary.txt
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:"gemm|attention|retrieve" -s 370 -c 13 -o $OUT/prof \
  python bench.py --quick --steps 2 --warmup 3 --no-cpu-baseline > $OUT/ncu_full_run.log 2>&1
python tools/ncu_summary.py $OUT/prof.ncu-rep $OUT/ncu_layer.txt $OUT/ncu_layer.json > /dev/null 2>&1; cat $OUT/ncu_layer.txt
ncu -i $OUT/prof.ncu-rep --page details --csv > $OUT/details.csv 2>/dev/null
python tools/ncu_details.py $OUT/details.csv > $OUT/details.txt 2>/dev/null
rm -f $OUT/details.csv
ls -la $OUT
