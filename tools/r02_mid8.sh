timeout 900 python -m pytest tests/test_engine_gpu.py tests/test_gemm_gpu.py -x -q > gpurun_out/mid8_tests.log 2>&1; tail -2 gpurun_out/mid8_tests.log
AB_VARIANTS=prev bash tools/r02_ab2.sh
AB_VARIANTS=prev bash tools/r02_ab2.sh
OUT=gpurun_out/r02end
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemm|attention|retrieve|route|fetch|head|scatter" -s 400 -c 120 --csv \
  --log-file $OUT/launches.csv python bench.py --quick --steps 3 --warmup 3 --no-cpu-baseline > $OUT/ncu_launch_run.log 2>&1
python tools/launch_summary.py $OUT/launches.csv $OUT/launches_summary.txt > /dev/null 2>&1; cat $OUT/launches_summary.txt
