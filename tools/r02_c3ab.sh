#!/usr/bin/env bash
# C3: generation tests, then the C3 line with the K-split decode GEMMs and without (same box)
OUT=gpurun_out/${1:-c3ab}
mkdir -p $OUT
HMI_DEBUG_PLAN=1 timeout 900 python -m pytest tests -m gpu -x -q -k "generate or lm or gpt or c3 or wide or token or decode" > $OUT/tests.log 2>&1; tail -3 $OUT/tests.log
grep "decode gemm plan" $OUT/tests.log | sort | uniq | head -20
for v in 1 0 1 0; do
  HMI_DEC_GEMM=$v timeout 600 python bench.py --config c3 --no-cpu-baseline > $OUT/c3_$v.json 2>$OUT/c3_$v.err
  python -c "import json; d=json.loads(open('$OUT/c3_$v.json').read().strip().splitlines()[-1]); print('dec_gemm=$v', round(d['value']), round(d['roofline']['step_ms'],4), round(d['roofline']['frac'],3)); [print('  ', k, round(v['ms_per_batch'],3)) for k,v in d['kernels'].items() if k.startswith('gemm')]"
done
