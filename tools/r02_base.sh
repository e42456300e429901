# round 2 (session 3): HEAD baseline — two bench lines and the GPU test suite
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
for r in 1 2; do
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/base_$r.json 2>>gpurun_out/base.err
python -c "import json; d=json.loads(open('gpurun_out/base_$r.json').read().strip().splitlines()[-1]); print('base', round(d['value']), round(d['ms_per_step'],3), d['e2e']['value'], {k: round(1e3*v['ms_per_launch'],1) for k,v in d['kernels'].items()}, d['clocks'])"
done
timeout 2400 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/pytest_gpu.log 2>&1
tail -30 gpurun_out/pytest_gpu.log
