# SPDX-License-Identifier: Apache-2.0
"""Soak run of the serving path: hBERT-base, `tenants` tenants through an HBM slot pool holding
half of them, `batches` mixed 256-request batches via the pipelined submit / wait API, with
adapter replacements, tenant migrations between two engines and table uploads interleaved.
Checks: every batch returns, no device error, pool residency within capacity, device memory
flat after warm-up, and a fixed probe batch scores identically at the start and the end.
    python tools/soak.py [tenants] [batches]"""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2504_17449_b200 import engine as E  # noqa: E402
from paper_2504_17449_b200.workload import CONFIGS, World  # noqa: E402

n_tenants = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
n_batches = int(sys.argv[2]) if len(sys.argv) > 2 else 1500
wl = CONFIGS["c2"]
world = World(wl)
mc = E.model_config(wl.hidden_size, wl.heads, wl.lower_layers, wl.higher_layers, wl.ffn_size,
                    wl.vocab_size, wl.mode, wl.max_fragment, wl.model_seed)
higher = E.generate_higher(mc)
layer_bytes = (wl.hidden_size * wl.r * 2 + wl.r + wl.hidden_size) * 4
tenants = list(range(n_tenants))
base = [E.generate_adapter(mc, wl.r, 1000 + t) for t in range(32)]


def engine():
    eng = E.GpuEngine(mc, higher, max_batch=wl.batch, max_seq=wl.seq, bottleneck=wl.r,
                      max_labels=wl.labels, pool_bytes=(n_tenants // 2) * wl.higher_layers * layer_bytes,
                      max_tasks=n_tenants, max_versions=len(world.tables) + 4)
    for t in world.tables:
        eng.upload_table(t["version"], t["parent"], t["key_len"], t["keys"], t["reps"])
    return eng


a, b = engine(), engine()
a.register_tasks(tenants, [base[t % 32] for t in tenants])
for t in tenants:
    w, bb = E.generate_head(wl.hidden_size, wl.labels, 2_000_000 + t)
    for e in (a, b):
        e.register_head(t, wl.head_kind, w, bb)
    a.bind_instance(t, world.tenant_version(t), t, t)
probe = world.requests(99, wl.batch, tenants=tenants[:wl.batch])
first = a.infer_batch(*probe).scores
free0 = None
t0 = time.perf_counter()
pending, done, migrated = [], 0, []
for k in range(n_batches):
    inst, toks, lens = world.requests(1000 + k % 64, wl.batch, tenants=tenants)
    inst = np.array([t for t in inst if t not in migrated] or [0], np.uint32)[:wl.batch]
    pending.append(a.submit_batch(inst, toks[:len(inst)], lens[:len(inst)]))
    if len(pending) >= 3:
        a.wait_batch(pending.pop(0))
        done += 1
    if k % 100 == 50:  # admin traffic between batches
        t = 1000 + (k // 100) % 500
        a.replace_task(t, base[(t + k) % 32])
        a.replace_task(t, base[t % 32])
        if t not in migrated and t >= wl.batch:
            a.migrate_task(b, t, keep_source=False)
            b.bind_instance(t, world.tenant_version(t), t, t)
            migrated.append(t)
    if k == 200:
        torch.cuda.synchronize()
        free0 = torch.cuda.mem_get_info()[0]
for p in pending:
    a.wait_batch(p)
    done += 1
a.synchronize()
wall = time.perf_counter() - t0
free1 = torch.cuda.mem_get_info()[0]
last = a.infer_batch(*probe).scores
st = a.pool_stats()
print(json.dumps({"tool": "soak", "tenants": n_tenants, "batches": done, "wall_s": round(wall, 2),
                  "req_per_s": round(done * wl.batch / wall), "migrated": len(migrated),
                  "pool_within_capacity": st["max_resident_bytes_seen"] <= st["capacity_bytes"],
                  "device_free_drift_mb": round((free0 - free1) / 2**20, 1) if free0 else None,
                  "probe_identical": bool(np.array_equal(first, last)), "pool": st}))
a.close()
b.close()
