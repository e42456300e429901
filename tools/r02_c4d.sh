for p in 0.5; do
timeout 900 python bench.py --config c4 --pool-fraction $p --no-cpu-baseline --steps 40 > gpurun_out/c4d_$p.json 2>>gpurun_out/c4d.err
python -c "import json; d=json.loads(open('gpurun_out/c4d_$p.json').read().strip().splitlines()[-1]); print('c4 $p', round(d['value']), round(d['ms_per_step'],3), d.get('swap'), d.get('h2d_gbps_per_rank'))"
done
tail -3 gpurun_out/c4d.err
