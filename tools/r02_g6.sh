# round 2: retrieval phase-2 variants + device readiness flags (fine mode)
timeout 900 python -m pytest -q -x tests/test_engine_gpu.py tests/test_parity_scale.py::test_c2_parity_1024_requests > gpurun_out/g6_tests.log 2>&1; tail -3 gpurun_out/g6_tests.log
for v in 0 1 2 3; do
HMI_RETR=$v timeout 600 python bench.py --no-cpu-baseline > gpurun_out/g6_retr$v.json 2>>gpurun_out/g6.err
python -c "import json; d=json.loads(open('gpurun_out/g6_retr$v.json').read().strip().splitlines()[-1]); print('retr $v', round(d['value']), round(d['ms_per_step'],3), 'retrieve us', round(1e3*d['kernels']['retrieve']['ms_per_launch'],1), d['clocks']['sm_mhz'])"
done
for m in fine coarse; do for p in 0.5 1.0; do
timeout 900 python bench.py --config c4 --pool-fraction $p --mode $m --no-cpu-baseline > gpurun_out/g6_c4_${m}_${p}.json 2>>gpurun_out/g6.err
python -c "import json; d=json.loads(open('gpurun_out/g6_c4_${m}_${p}.json').read().strip().splitlines()[-1]); print('$m $p', round(d['value']), round(d['ms_per_step'],3), d['clocks']['sm_mhz'], (d.get('swap') or {}).get('compute_idle_ms_per_step'))"
done; done
tail -5 gpurun_out/g6.err
