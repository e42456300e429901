#!/usr/bin/env bash
# End-of-session check at HEAD: GPU suite, smoke, C2 line, C3 line + its ncu launch list
OUT=gpurun_out/${1:-end}
mkdir -p $OUT
HMI_PARITY_OUT=$OUT/parity timeout 2400 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.txt 2>&1; tail -2 $OUT/pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1; tail -1 $OUT/smoke.txt
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; tail -c 300 $OUT/bench.json; echo
timeout 600 python bench.py --config c3 --no-cpu-baseline > $OUT/c3.json 2>$OUT/c3.err; tail -c 200 $OUT/c3.json; echo
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 600 --csv \
  --log-file $OUT/c3_launches.csv python bench.py --config c3 --steps 1 --warmup 3 --no-cpu-baseline > $OUT/ncu_run.log 2>&1
python tools/launch_summary.py $OUT/c3_launches.csv $OUT/c3_launches_summary.txt > /dev/null 2>&1; cat $OUT/c3_launches_summary.txt
