# round 2: C4 mode comparison, bf16 C2 line, C3 line with the decode roofline, PLOT builder line
for m in coarse fine; do for p in 0.5 1.0; do
timeout 900 python bench.py --config c4 --pool-fraction $p --mode $m --no-cpu-baseline --steps 20 > gpurun_out/c4_${m}_${p}.json 2>>gpurun_out/g5.err
python -c "import json; d=json.loads(open('gpurun_out/c4_${m}_${p}.json').read().strip().splitlines()[-1]); print('$m $p', round(d['value']), round(d['ms_per_step'],3), d['clocks'], d.get('swap'))"
done; done
timeout 600 python bench.py --precision 1 --no-cpu-baseline > gpurun_out/c2_bf16.json 2>>gpurun_out/g5.err; tail -c 300 gpurun_out/c2_bf16.json
timeout 900 python bench.py --config c3 --steps 5 --warmup 3 > gpurun_out/c3.json 2>>gpurun_out/g5.err; tail -c 1500 gpurun_out/c3.json
timeout 900 python bench.py --config plot --steps 3 --warmup 3 > gpurun_out/plot.json 2>>gpurun_out/g5.err; tail -c 800 gpurun_out/plot.json
tail -20 gpurun_out/g5.err
