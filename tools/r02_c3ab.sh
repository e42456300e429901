#!/usr/bin/env bash
# C3: generation / lm-head tests, then the C3 line twice with its per-class profile
OUT=gpurun_out/${1:-c3ab}
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q -k "generate or lm or gpt or c3 or wide or token or decode" > $OUT/tests.log 2>&1; tail -3 $OUT/tests.log
for i in 1 2; do
  timeout 600 python bench.py --config c3 --no-cpu-baseline > $OUT/c3_$i.json 2>$OUT/c3_$i.err
  python -c "import json; d=json.loads(open('$OUT/c3_$i.json').read().strip().splitlines()[-1]); print(round(d['value']), round(d['roofline']['step_ms'],4), round(d['roofline']['frac'],3)); [print('  ', k, round(v['ms_per_batch'],3)) for k,v in d['kernels'].items()]"
done
