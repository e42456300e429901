# SPDX-License-Identifier: Apache-2.0
"""Summarise an `ncu --set full` capture of one C2 layer into profiles/ (text + json).

The capture (tools/profile.sh) holds, in launch order: retrieve, then higher
layers 0 and 1 (gemm_qkv, attention, adapter_down (tenant-grouped down
projection from ctx), gemm_oproj (O projection + the tenants' up projections
+ residual + LN statistics), gemm_ffn1, gemm_ffn2 each; layer 1's QKV is the
LN-folded variant). Keys without a suffix are layer 1 (the steady-state layer).
"""
import csv
import io
import json
import subprocess
import sys

# LayerNorm folded (default engine mode): retrieval, then layer 0 and layer 1
LAYER = ["gemm_qkv", "attention", "adapter_down", "gemm_oproj", "gemm_ffn1", "gemm_ffn2"]
ORDER = ["retrieve"] + [f"{k}@L0" for k in LAYER] + LAYER
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
           "launch__grid_size", "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
           "lts__throughput.avg.pct_of_peak_sustained_elapsed",
           "smsp__cycles_active.avg", "sm__cycles_elapsed.avg.per_second"]


def main(rep, out_txt, out_json):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    ix = {h: i for i, h in enumerate(hdr)}
    summary = {"source": rep, "kernels": {}}
    lines = [f"{'class':14s} {'kernel':44s} {'us':>8s} {'DRAM MB':>9s} {'dram%':>6s} {'tensor%':>8s} {'regs':>5s} {'grid':>6s}"]
    for name, row in zip(ORDER, data):
        def g(m):
            return row[ix[m]] if m in ix else ""
        t = float(g("gpu__time_duration.sum"))
        tu = units[ix["gpu__time_duration.sum"]]
        t_us = t / 1000 if tu == "nsecond" else (t * 1000 if tu == "msecond" else t)
        bu = units[ix["dram__bytes_read.sum"]]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(bu, 1)
        rd = float(g("dram__bytes_read.sum")) * scale
        wr = float(g("dram__bytes_write.sum")) * scale
        summary["kernels"][name] = {
            "kernel": row[ix["Kernel Name"]], "time_us": t_us, "dram_bytes": rd + wr,
            "dram_read_bytes": rd, "dram_write_bytes": wr,
            "dram_pct": float(g("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed") or 0),
            "tensor_pct": float(g("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed") or 0),
            "registers": int(float(g("launch__registers_per_thread") or 0)),
            "grid": int(float(g("launch__grid_size") or 0)),
        }
        k = summary["kernels"][name]
        lines.append(f"{name:14s} {k['kernel'][:44]:44s} {t_us:8.1f} {(rd + wr) / 1e6:9.1f} "
                     f"{k['dram_pct']:6.1f} {k['tensor_pct']:8.1f} {k['registers']:5d} {k['grid']:6d}")
    open(out_txt, "w").write("\n".join(lines) + "\n")
    json.dump(summary, open(out_json, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main(*sys.argv[1:4])
