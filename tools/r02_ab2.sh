# same-box A/B of experimental libraries in abtest/ against the working tree's library
for r in 1 2; do
for v in new ${AB_VARIANTS:-novec}; do
if [ $v = new ]; then unset HMI_LIB_PATH; else export HMI_LIB_PATH=$PWD/abtest/$v.so; fi
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/ab_${v}_$r.json 2>>gpurun_out/ab.err
python -c "import json; d=json.loads(open('gpurun_out/ab_${v}_$r.json').read().strip().splitlines()[-1]); print('$v', round(d['value']), round(d['ms_per_step'],3), {k: round(1e3*v['ms_per_launch'],1) for k,v in d['kernels'].items() if k not in ('h2d_inputs','route','head')}, d['clocks']['reasons'])"
done; done
tail -3 gpurun_out/ab.err
