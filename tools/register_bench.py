# SPDX-License-Identifier: Apache-2.0
"""Adapter registration throughput ("10k adapters need fast load"):
C2 adapters (d 768, r 64, 6 higher layers) registered one call at a time, in bulk on host
threads, and in bulk from ADP1 files (page cache warm).   python tools/register_bench.py [n]"""
import json
import os
import sys
import tempfile
import time

sys.path.insert(0, ".")
from paper_2504_17449_b200 import engine as E  # noqa: E402
from paper_2504_17449_b200 import plot  # noqa: E402
from paper_2504_17449_b200.workload import CONFIGS  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
wl = CONFIGS["c2"]
mc = E.model_config(wl.hidden_size, wl.heads, wl.lower_layers, wl.higher_layers, wl.ffn_size,
                    wl.vocab_size, wl.mode, wl.max_fragment, wl.model_seed)
higher = E.generate_higher(mc)
base = [E.generate_adapter(mc, wl.r, 1000 + t) for t in range(16)]
adapters = [base[t % 16] for t in range(n)]
tmp = tempfile.mkdtemp()
paths = []
for t in range(16):
    p = os.path.join(tmp, f"a{t}.adp1")
    plot.save_adp1(p, f"t{t}", base[t], wl.hidden_size, wl.r)
    paths.append(p)
paths = [paths[t % 16] for t in range(n)]
res = {}
for name in ("one_by_one", "bulk_arrays", "bulk_files"):
    eng = E.GpuEngine(mc, higher, max_batch=8, max_seq=128, bottleneck=wl.r, max_labels=8,
                      max_tasks=n, max_versions=2)
    eng.register_tasks(range(n), adapters)  # warm the pinned store, then free it
    for t in range(n):
        eng.unregister_task(t)
    t0 = time.perf_counter()
    if name == "one_by_one":
        for t in range(n):
            eng.register_task(t, adapters[t])
    elif name == "bulk_arrays":
        eng.register_tasks(range(n), adapters)
    else:
        eng.register_task_files(range(n), paths)
    dt = time.perf_counter() - t0
    res[name] = {"ms_per_task": dt / n * 1e3, "tasks_per_s": n / dt}
    eng.close()
print(json.dumps({"tool": "register", "tasks": n, "f32_bytes_per_task":
                  int(adapters[0].nbytes), "cores": os.cpu_count(), "results": res}))
