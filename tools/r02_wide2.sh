# wide / epilogue-skipped variants (timing only; the no-epilogue builds compute nothing useful)
for v in new ${W2_VARIANTS:-wide widenoepi pairnoepi}; do
if [ $v = new ]; then unset HMI_LIB_PATH; else export HMI_LIB_PATH=$PWD/abtest/$v.so; fi
timeout 300 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/w2_${v}.json 2>>gpurun_out/w2.err
python -c "import json; d=json.loads(open('gpurun_out/w2_${v}.json').read().strip().splitlines()[-1]); print('$v', round(d['value']), round(d['ms_per_step'],3), {k: round(1e3*v['ms_per_launch'],1) for k,v in d['kernels'].items() if k in ('gemm_qkv','gemm_ffn1','gemm_ffn2','gemm_oproj')})"
done
tail -3 gpurun_out/w2.err
