# round 2: full GPU suite, C2 line, C4 pool 0.5 vs 1.0 (fine), C3 line
timeout 2400 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/pytest_gpu.log 2>&1; tail -14 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/full_c2.json 2>>gpurun_out/full.err
python -c "import json; d=json.loads(open('gpurun_out/full_c2.json').read().strip().splitlines()[-1]); print('c2', round(d['value']), round(d['ms_per_step'],3), round(d['e2e']['value']), d['roofline']['frac_of_burst'], d['roofline'].get('step_tensor_frac'))"
for p in 1.0 0.5 1.0 0.5; do
timeout 900 python bench.py --config c4 --pool-fraction $p --no-cpu-baseline --steps 60 > gpurun_out/full_c4_$p.json 2>>gpurun_out/full.err
python -c "import json; d=json.loads(open('gpurun_out/full_c4_$p.json').read().strip().splitlines()[-1]); print('c4 $p', round(d['value']), round(d['ms_per_step'],3), d['clocks']['reasons'], d.get('swap'))"
done
timeout 900 python bench.py --config c3 --no-cpu-baseline > gpurun_out/full_c3.json 2>>gpurun_out/full.err
python -c "import json; d=json.loads(open('gpurun_out/full_c3.json').read().strip().splitlines()[-1]); print('c3', round(d['value']), round(d['ms_per_step'],3), d['roofline']['frac'], d['roofline']['step_ms'])"
tail -3 gpurun_out/full.err
