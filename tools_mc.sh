timeout 300 python tools_numa_probe.py 2>&1 | grep -v Warn
timeout 240 python tools_gemm_sweep.py --mc 2>&1 | grep -v Warn; echo "sweep rc $?"
