for g in 16 32 64; do
HMI_GATHER_CTAS=$g timeout 900 python bench.py --config c4 --pool-fraction 0.5 --no-cpu-baseline --steps 40 > gpurun_out/c4c_$g.json 2>>gpurun_out/c4c.err
python -c "import json; d=json.loads(open('gpurun_out/c4c_$g.json').read().strip().splitlines()[-1]); s=d.get('swap'); print('c4 0.5 ctas $g', round(d['value']), round(d['ms_per_step'],3), round(s['io_busy_ms_per_step'],2), round(s['compute_busy_ms_per_step'],2), round(s['io_hidden_frac'],3))"
done
tail -3 gpurun_out/c4c.err
