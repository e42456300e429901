# C3 decode work: generation / lm-head tests, then the C3 line with its per-class profile
timeout 900 python -m pytest tests -m gpu -x -q -k "generate or lm or gpt or c3 or wide or token" > gpurun_out/c3_tests.log 2>&1; tail -2 gpurun_out/c3_tests.log
timeout 600 python bench.py --config c3 --no-cpu-baseline > gpurun_out/c3p.json 2>gpurun_out/c3p.err; tail -2 gpurun_out/c3p.err
python -c "import json; d=json.loads(open('gpurun_out/c3p.json').read().strip().splitlines()[-1]); print(round(d['value']), round(d['roofline']['step_ms'],4), round(d['roofline']['frac'],3), d['roofline']['prefill_ms']); [print(k, round(v['ms_per_batch'],3), v['launches_per_batch']) for k,v in d['kernels'].items()]"
