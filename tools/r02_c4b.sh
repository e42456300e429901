timeout 900 python -m pytest tests/test_engine_gpu.py -x -q -k "swap or pool or pipeline or stage or submit" > gpurun_out/c4b_tests.log 2>&1; tail -2 gpurun_out/c4b_tests.log
for p in 1.0 0.5 1.0 0.5; do
timeout 900 python bench.py --config c4 --pool-fraction $p --no-cpu-baseline --steps 60 > gpurun_out/c4b_$p.json 2>>gpurun_out/c4b.err
python -c "import json; d=json.loads(open('gpurun_out/c4b_$p.json').read().strip().splitlines()[-1]); print('c4 $p', round(d['value']), round(d['ms_per_step'],3), d['clocks']['reasons'], d.get('swap'))"
done
tail -3 gpurun_out/c4b.err
