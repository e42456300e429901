# SPDX-License-Identifier: Apache-2.0
"""Tenant migration cost: hBERT-base adapters (C2, r = 64, 12 layers)
moved between two engines by export / import (device-to-device slot copies; on one GPU the
"peer" is the same device, so this measures the copy path and bookkeeping, not NVLink) against
the PCIe path a migration would otherwise take: register_task on the destination followed by
the H2D residency load of its first batch.   python tools/migrate_bench.py [tasks]"""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2504_17449_b200 import engine as E  # noqa: E402
from paper_2504_17449_b200.workload import CONFIGS, World  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
wl = CONFIGS["c2"]
world = World(wl)
mc = E.model_config(wl.hidden_size, wl.heads, wl.lower_layers, wl.higher_layers, wl.ffn_size,
                    wl.vocab_size, wl.mode, wl.max_fragment, wl.model_seed)
higher = E.generate_higher(mc)
adapters = [E.generate_adapter(mc, wl.r, 1000 + t) for t in range(n)]


def engine():
    eng = E.GpuEngine(mc, higher, max_batch=wl.batch, max_seq=wl.seq, bottleneck=wl.r,
                      max_labels=wl.labels, max_tasks=n, max_versions=len(world.tables) + 1)
    for t in world.tables:
        eng.upload_table(t["version"], t["parent"], t["key_len"], t["keys"], t["reps"])
    # warm the pinned host store (256 MB chunks, recycled blocks): steady state, not first-touch
    for t in range(n):
        eng.register_task(t, adapters[t])
    for t in range(n):
        eng.unregister_task(t)
    return eng


src, dst = engine(), engine()
for t in range(n):
    src.register_task(t, adapters[t])
for t in range(n):  # all resident at the source
    src.export_task(t)
    src.release_export(t)
src.synchronize()

phase = {"export": 0.0, "import": 0.0, "release": 0.0}
moved = 0
t0 = time.perf_counter()
for t in range(n):  # GpuEngine.migrate_task, phase by phase
    a = time.perf_counter()
    ex = src.export_task(t)
    b = time.perf_counter()
    moved += dst.import_task(t, ex)
    c = time.perf_counter()
    src.release_export(t, drop=True)
    phase["export"] += b - a
    phase["import"] += c - b
    phase["release"] += time.perf_counter() - c
dst.synchronize()
mig = time.perf_counter() - t0

pcie = engine()
t0 = time.perf_counter()
for t in range(n):
    pcie.register_task(t, adapters[t])
    pcie.export_task(t)  # forces the H2D residency load of every layer, as a first batch would
pcie.synchronize()
h2d = time.perf_counter() - t0
line = {"tool": "migrate", "tasks": n, "bytes_per_task": moved // n,
        "peer_ms_per_task": mig / n * 1e3,
        "phase_ms_per_task": {k: v / n * 1e3 for k, v in phase.items()}, "peer_gbps": moved / mig / 1e9,
        "register_h2d_ms_per_task": h2d / n * 1e3, "register_h2d_gbps": moved / h2d / 1e9,
        "note": "one GPU: peer copy is same-device D2D; includes export/import bookkeeping"}
print(json.dumps(line))
for e in (src, dst, pcie):
    e.close()
