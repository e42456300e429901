# SPDX-License-Identifier: Apache-2.0
"""Pipeline-mode ablation with StageTrace (paper
Table 12): hBERT-base, `n_tenants` tenants whose adapters swap through an HBM slot pool holding
`pool` of them, 256-request batches, sync / coarse / fine. Per mode: requests/s over the
makespan of the traced batches, io (adapter H2D) and compute busy time, and how much of the io
time overlaps compute.   python tools/stage_ablation.py [n_tenants] [pool] [batches]"""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2504_17449_b200 import engine as E  # noqa: E402
from paper_2504_17449_b200.workload import CONFIGS, World  # noqa: E402

n_tenants = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
pool = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
n_batches = int(sys.argv[3]) if len(sys.argv) > 3 and sys.argv[3].isdigit() else 12
wl = CONFIGS["c2"]
world = World(wl)
mc = E.model_config(wl.hidden_size, wl.heads, wl.lower_layers, wl.higher_layers, wl.ffn_size,
                    wl.vocab_size, wl.mode, wl.max_fragment, wl.model_seed)
higher = E.generate_higher(mc)
tenants = list(range(n_tenants))
adapters = {t: E.generate_adapter(mc, wl.r, 1000 + t) for t in tenants}
heads = {t: E.generate_head(wl.hidden_size, wl.labels, 2_000_000 + t) for t in tenants}
ref_layer_bytes = (wl.hidden_size * wl.r * 2 + wl.r + wl.hidden_size) * 4
batches = [world.requests(7000 + s, wl.batch, tenants=tenants) for s in range(n_batches + 2)]


def union(iv):
    iv = sorted(iv)
    out = []
    for a, b in iv:
        if out and a <= out[-1][1]:
            out[-1][1] = max(out[-1][1], b)
        else:
            out.append([a, b])
    return out


def overlap(x, y):
    tot, j = 0.0, 0
    for a, b in x:
        for c, d in y:
            tot += max(0.0, min(b, d) - max(a, c))
    return tot


rows = {}
for name, mode in (("sync", E.MODE_SYNC), ("coarse", E.MODE_COARSE), ("fine", E.MODE_FINE)):
    eng = E.GpuEngine(mc, higher, max_batch=wl.batch, max_seq=wl.seq, bottleneck=wl.r,
                      max_labels=wl.labels, pipeline_mode=mode,
                      pool_bytes=int(pool * n_tenants) * wl.higher_layers * ref_layer_bytes,
                      max_tasks=n_tenants, max_versions=len(world.tables) + 1)
    for t in world.tables:
        eng.upload_table(t["version"], t["parent"], t["key_len"], t["keys"], t["reps"])
    for t in tenants:
        eng.register_task(t, adapters[t])
        eng.register_head(t, wl.head_kind, *heads[t])
        eng.bind_instance(t, world.tenant_version(t), t, t)
    for inst, toks, lens in batches[:2]:  # warm-up (fills the pool)
        eng.infer_batch(inst, toks, lens)
    eng.synchronize()
    eng.trace(True)
    t0 = time.perf_counter()
    ts = []
    for inst, toks, lens in batches[2:]:
        ts.append(eng.submit_batch(inst, toks, lens))
        if len(ts) >= 3:
            eng.wait_batch(ts.pop(0))
    for t in ts:
        eng.wait_batch(t)
    wall = time.perf_counter() - t0
    recs = eng.stage_trace()
    eng.trace(False)
    st = eng.pool_stats()
    eng.close()
    dev = [r for r in recs if r["worker"] != "cpu"]
    span = max(r["end_ms"] for r in dev) - min(r["start_ms"] for r in dev)
    io = union([(r["start_ms"], r["end_ms"]) for r in recs if r["worker"] == "io"])
    comp = union([(r["start_ms"], r["end_ms"]) for r in recs if r["worker"] == "compute"])
    io_busy = sum(b - a for a, b in io)
    comp_busy = sum(b - a for a, b in comp)
    rows[name] = {
        "req_per_s": n_batches * wl.batch / (span / 1e3), "makespan_ms": span,
        "wall_req_per_s": n_batches * wl.batch / wall,
        "io_busy_ms": io_busy, "compute_busy_ms": comp_busy,
        "io_hidden_frac": overlap(io, comp) / io_busy if io_busy > 0 else 1.0,
    }
    print(name, json.dumps({k: round(v, 3) for k, v in rows[name].items()}), flush=True)
    if "--timeline" in sys.argv:
        t0 = min(r["start_ms"] for r in dev)
        for bt in sorted({r["batch"] for r in recs})[:6]:
            io_b = [r for r in recs if r["batch"] == bt and r["worker"] == "io"]
            cp_b = [r for r in recs if r["batch"] == bt and r["worker"] == "compute"]
            host = [r for r in recs if r["batch"] == bt and r["worker"] == "cpu"]
            print(f"  batch {bt}: host {host[0]['start_ms'] - t0:7.2f}-{host[0]['end_ms'] - t0:7.2f}  "
                  f"io {min(r['start_ms'] for r in io_b) - t0:7.2f}-{max(r['end_ms'] for r in io_b) - t0:7.2f}  "
                  f"compute {min(r['start_ms'] for r in cp_b) - t0:7.2f}-{max(r['end_ms'] for r in cp_b) - t0:7.2f}")
print(json.dumps({"ablation": "pipeline modes with StageTrace", "tenants": n_tenants,
                  "pool_fraction": pool, "batches": n_batches, "batch": wl.batch, "modes": rows,
                  "fine_over_sync": rows["fine"]["req_per_s"] / rows["sync"]["req_per_s"]}))
