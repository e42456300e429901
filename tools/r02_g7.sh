# round 2: retrieval variants (per-kernel event time), interleaved C4 A/B with 60 timed steps
for v in 1 4 5 1 4; do
HMI_RETR=$v timeout 600 python bench.py --no-cpu-baseline > gpurun_out/g7_retr$v.json 2>>gpurun_out/g7.err
python -c "import json; d=json.loads(open('gpurun_out/g7_retr$v.json').read().strip().splitlines()[-1]); print('retr $v', round(d['value']), round(d['ms_per_step'],3), 'retrieve us', round(1e3*d['kernels']['retrieve']['ms_per_launch'],1), d['clocks']['sm_mhz'])"
done
for r in 1 2; do for m in fine coarse; do for p in 1.0 0.5; do
timeout 900 python bench.py --config c4 --pool-fraction $p --mode $m --no-cpu-baseline --steps 60 > gpurun_out/g7_c4_${m}_${p}_$r.json 2>>gpurun_out/g7.err
python -c "import json; d=json.loads(open('gpurun_out/g7_c4_${m}_${p}_$r.json').read().strip().splitlines()[-1]); print('$m $p', round(d['value']), round(d['ms_per_step'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'], (d.get('swap') or {}).get('compute_idle_ms_per_step'))"
done; done; done
tail -5 gpurun_out/g7.err
