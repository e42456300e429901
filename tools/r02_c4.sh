# C4 swap diagnostics (round 2): host submit times and device step at pool 0.5 / 1.0, then the bench trace
timeout 600 python tools/c4_diag.py fine 0.5 > gpurun_out/c4diag_05.txt 2>&1; cat gpurun_out/c4diag_05.txt
timeout 600 python tools/c4_diag.py fine 1.0 > gpurun_out/c4diag_10.txt 2>&1; cat gpurun_out/c4diag_10.txt
timeout 900 python bench.py --config c4 --pool-fraction 0.5 --no-cpu-baseline > gpurun_out/b4_c4_05.json 2>gpurun_out/b4_c4.err; tail -c 700 gpurun_out/b4_c4_05.json
