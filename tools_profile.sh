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
# per batch: retrieve + 7 GEMM/attention launches per layer (LN folded); skip 2 batches
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:"gemm|attention|retrieve" -s 86 -c 15 -o $OUT/prof \
  python bench.py --quick --steps 2 --warmup 3 --no-cpu-baseline > $OUT/ncu_full_run.log 2>&1
ls -la $OUT
