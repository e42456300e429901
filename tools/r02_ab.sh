# same-box A/B: abtest/head.so (previous commit, per-copy swaps) vs the working tree's library
for r in 1 2 3; do
for v in head new; do
if [ $v = head ]; then export HMI_LIB_PATH=$PWD/abtest/head.so; else unset HMI_LIB_PATH; fi
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/ab_${v}_$r.json 2>>gpurun_out/ab.err
python -c "import json; d=json.loads(open('gpurun_out/ab_${v}_$r.json').read().strip().splitlines()[-1]); print('$v', round(d['value']), round(d['ms_per_step'],3), round(d['e2e']['value']), {k: round(1e3*v['ms_per_launch'],1) for k,v in d['kernels'].items()}, d['clocks']['reasons'])"
done; done
tail -3 gpurun_out/ab.err
