#!/usr/bin/env bash
# GEMM shape sweep (ours vs cuBLAS) + ncu L2/tensor metrics of the cta_group::2 launches.
OUT=gpurun_out/${1:-gemm_l2}
mkdir -p $OUT
timeout 600 python tools/gemm_sweep.py > $OUT/sweep.txt 2>&1; echo "sweep rc $?"; cat $OUT/sweep.txt
M=gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__m_xbar2l1tex_read_bytes.sum,sm__cycles_elapsed.avg.per_second,lts__cycles_elapsed.avg.per_second
timeout 900 ncu --metrics $M --clock-control none -k regex:gemm --csv --log-file $OUT/ncu_l2.csv \
  python tools/gemm_sweep.py --ncu > $OUT/ncu_run.log 2>&1; echo "ncu rc $?"
python3 - $OUT/ncu_l2.csv <<'PY'
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = None
for r in rows:
    if r and r[0] == "ID":
        hdr = r; continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        print(d["ID"], d["Kernel Name"][:40], d["Metric Name"], d["Metric Unit"], d["Metric Value"])
PY
