#!/usr/bin/env bash
# One GPU call: parity tests, the bench line, the ncu launch list and one
# `ncu --set full` capture of retrieval + two higher layers of the C2 step.
set -x
OUT=gpurun_out/${1:-r01}
mkdir -p $OUT
make -s oracle >/dev/null
timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -5 > $OUT/pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 400 -c 120 --csv \
  --log-file $OUT/launches.csv python bench.py --quick --steps 3 --warmup 3 --no-cpu-baseline > $OUT/ncu_launch_run.log 2>&1
# per batch: retrieve + 6 launches per layer (QKV, attention, O, fused adapter, FFN1, FFN2);
# skip the 10 warm-up batches, capture retrieval + layers 0 and 1 of the next one
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:"gemm|attention|retrieve|adapter" -s 370 -c 13 -o $OUT/prof \
  python bench.py --quick --steps 2 --warmup 3 --no-cpu-baseline > $OUT/ncu_full_run.log 2>&1
python tools/ncu_summary.py $OUT/prof.ncu-rep $OUT/ncu_layer.txt $OUT/ncu_layer.json > /dev/null 2>&1
ncu -i $OUT/prof.ncu-rep --page details --csv > $OUT/details.csv 2>/dev/null
python tools/ncu_details.py $OUT/details.csv > $OUT/details.txt 2>/dev/null
python tools/launch_summary.py $OUT/launches.csv $OUT/launches_summary.txt > /dev/null 2>&1
ls -la $OUT
