# round 2: O projection with tenant up-projection K blocks (kEpiExt) + folded down projection
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests/test_engine_gpu.py -x -q > gpurun_out/ext_engine.log 2>&1; tail -15 gpurun_out/ext_engine.log
for r in 1 2; do
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/ext_$r.json 2>>gpurun_out/ext.err
python -c "import json; d=json.loads(open('gpurun_out/ext_$r.json').read().strip().splitlines()[-1]); print('ext', round(d['value']), round(d['ms_per_step'],3), d['e2e']['value'], {k: round(1e3*v['ms_per_launch'],1) for k,v in d['kernels'].items()}, d['clocks'])"
done
tail -5 gpurun_out/ext.err
timeout 2400 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/pytest_gpu.log 2>&1
tail -30 gpurun_out/pytest_gpu.log
