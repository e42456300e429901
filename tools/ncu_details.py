# SPDX-License-Identifier: Apache-2.0
"""Key metrics per kernel from an `ncu --page details --csv` export: python tools/ncu_details.py details.csv"""
import csv
import sys

WANT = ["Duration", "DRAM Throughput", "Memory Throughput", "L2 Cache Throughput", "L1/TEX Cache Throughput",
        "Compute (SM) Throughput", "Registers Per Thread", "Achieved Occupancy", "SM Frequency",
        "One or More Eligible", "No Eligible", "Issued Warp Per Scheduler", "Warp Cycles Per Issued Instruction",
        "Executed Ipc Active", "Grid Size", "Mem Busy", "Max Bandwidth", "Mem Pipes Busy"]
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[0]
ix = {h: i for i, h in enumerate(hdr)}
cur = None
for r in rows[1:]:
    if len(r) <= ix["Metric Value"] or r[ix["Metric Name"]] not in WANT:
        continue
    key = (r[ix["ID"]], r[ix["Kernel Name"]][:60])
    if key != cur:
        cur = key
        print(f"--- [{key[0]}] {key[1]}")
    print(f"    {r[ix['Metric Name']]:36s} {r[ix['Metric Value']]:>12s} {r[ix['Metric Unit']]}")
