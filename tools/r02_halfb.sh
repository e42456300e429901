# experiment: pair GEMMs loading half of each B tile (wrong results; per-kernel time only)
for r in 1 2; do
for v in new halfb; do
if [ $v = new ]; then unset HMI_LIB_PATH; else export HMI_LIB_PATH=$PWD/abtest/$v.so; fi
timeout 300 python bench.py --no-cpu-baseline --quick > gpurun_out/hb_${v}_$r.json 2>>gpurun_out/hb.err
python -c "import json; d=json.loads(open('gpurun_out/hb_${v}_$r.json').read().strip().splitlines()[-1]); print('$v', round(d['value']), round(d['ms_per_step'],3))"
done; done
tail -3 gpurun_out/hb.err
