# SPDX-License-Identifier: Apache-2.0
"""PLT1 ingest throughput: a C2-width (d = 768) branch table of
`rows` rep rows written as PLT1, then uploaded into a GPU engine by the streamed path
(hmi_gpu_upload_plt1: pinned chunks shipped whole, rows scattered on the device) and by the
host path (hmi_plot_table_load into host memory, then hmi_gpu_upload_plot_table). The file is
in the page cache (just written) for both: this measures the ingest, not the disk.
    python tools/ingest_bench.py [rows] [dir]"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2504_17449_b200 import engine as E  # noqa: E402
from paper_2504_17449_b200 import plot  # noqa: E402

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 600_000
out_dir = sys.argv[2] if len(sys.argv) > 2 else "/tmp"
d, vocab = 768, 30522
mc = E.model_config(d, 12, 6, 6, 3072, vocab, 0, 3, 1)
rng = np.random.default_rng(0)
n = rows // 2
kl = np.full(n, 2, np.uint32)
keys = np.zeros((n, 3), np.uint32)
keys[:, 0] = np.arange(n) // vocab
keys[:, 1] = np.arange(n) % vocab
reps = rng.standard_normal((2 * n, d), dtype=np.float32)
table = {"key_len": kl, "keys": keys, "freq": np.ones(n, np.uint64), "reps": reps}
path = os.path.join(out_dir, "ingest_bench.plt1")
plot.save_plt1(table, path, 1, 0, "bench", 5000)
size = os.path.getsize(path)
root = {"key_len": np.ones(vocab, np.uint32),
        "keys": np.stack([np.arange(vocab), np.zeros(vocab), np.zeros(vocab)], 1).astype(np.uint32),
        "reps": np.zeros((vocab, d), np.float32)}
higher = E.generate_higher(mc)
res = {}
for name, streamed in (("host_load_then_upload", False), ("streamed", True),
                       ("host_load_then_upload_2", False), ("streamed_2", True)):
    eng = E.GpuEngine(mc, higher, max_batch=8, max_seq=128, bottleneck=64, max_labels=8,
                      max_tasks=1, max_versions=4)
    eng.upload_table(0, 0xFFFFFFFF, root["key_len"], root["keys"], root["reps"])
    eng.synchronize()
    t0 = time.perf_counter()
    eng.upload_plt1(path, streamed=streamed)
    eng.synchronize()
    dt = time.perf_counter() - t0
    res[name] = {"s": dt, "GB_per_s": size / dt / 1e9}
    eng.close()
os.remove(path)
print(json.dumps({"tool": "ingest", "file_bytes": size, "rows": 2 * n, "entries": n, "d": d,
                  "results": res,
                  "note": "file in page cache; wall time of upload_plt1 incl. hash build + commit"}))
