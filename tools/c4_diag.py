# SPDX-License-Identifier: Apache-2.0
"""C4 swap diagnostics: host submit time per batch, device step time, bytes copied per batch,
and a copy-only bandwidth probe (pinned host -> HBM slots).  python tools/c4_diag.py [mode]"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2504_17449_b200 import engine as E  # noqa: E402
from paper_2504_17449_b200.workload import CONFIGS, World  # noqa: E402

mode_name = sys.argv[1] if len(sys.argv) > 1 else "fine"
frac = float(sys.argv[2]) if len(sys.argv) > 2 else 0.6
wl = CONFIGS["c4"]
world = World(wl)
mc = E.model_config(wl.hidden_size, wl.heads, wl.lower_layers, wl.higher_layers, wl.ffn_size,
                    wl.vocab_size, wl.mode, wl.max_fragment, wl.model_seed)
higher = E.generate_higher(mc)
tenants = list(range(wl.n_tenants))
ref_layer_bytes = (wl.hidden_size * wl.r * 2 + wl.r + wl.hidden_size) * 4
pool_bytes = int(frac * len(tenants)) * wl.higher_layers * ref_layer_bytes
mode = {"sync": E.MODE_SYNC, "coarse": E.MODE_COARSE, "fine": E.MODE_FINE}[mode_name]
eng = E.GpuEngine(mc, higher, device=0, precision=0, max_batch=wl.batch, max_seq=wl.seq,
                  bottleneck=wl.r, max_labels=wl.labels, pipeline_mode=mode, pool_bytes=pool_bytes,
                  max_tasks=wl.n_tenants, max_versions=len(world.tables) + 1)
for t in world.tables:
    eng.upload_table(t["version"], t["parent"], t["key_len"], t["keys"], t["reps"])
t0 = time.perf_counter()
for t in tenants:
    eng.register_task(t, E.generate_adapter(mc, wl.r, 1000 + t))
    w, b = E.generate_head(wl.hidden_size, wl.labels, 2_000_000 + t)
    eng.register_head(t, wl.head_kind, w, b)
    eng.bind_instance(t, world.tenant_version(t), t, t)
print(f"register {len(tenants)} tenants: {time.perf_counter() - t0:.1f} s", flush=True)
N = 24
batches = [world.requests(5000 + s, wl.batch, tenants=tenants) for s in range(N)]
dev = torch.device("cuda", 0)
d_tok = [torch.from_numpy(b[1].astype(np.int32)).to(dev) for b in batches]
d_len = [torch.from_numpy(b[2].astype(np.int32)).to(dev) for b in batches]
d_scores = torch.zeros((wl.batch, wl.labels), dtype=torch.float32, device=dev)
d_labels = torch.zeros((wl.batch,), dtype=torch.int32, device=dev)
for c in range(0, len(tenants), wl.batch):  # fill the pool
    chunk = np.array(tenants[c:c + wl.batch], np.uint32)
    _, toks, lens = world.requests(77 + c, len(chunk), tenants=chunk)
    eng.infer_batch(chunk, toks, lens)
eng.synchronize()
stream = torch.cuda.ExternalStream(eng.stream, device=dev)
st0 = eng.pool_stats()
host = []
a = torch.cuda.Event(enable_timing=True)
b = torch.cuda.Event(enable_timing=True)
a.record(stream)
w0 = time.perf_counter()
for i in range(N):
    h0 = time.perf_counter()
    inst, _, lens = batches[i]
    eng.infer_batch_device(inst, d_tok[i].data_ptr(), wl.seq, d_len[i].data_ptr(), int(lens.max()),
                           d_scores.data_ptr(), d_labels.data_ptr())
    host.append(time.perf_counter() - h0)
b.record(stream)
eng.synchronize()
torch.cuda.synchronize()
wall = time.perf_counter() - w0
st1 = eng.pool_stats()
dev_ms = a.elapsed_time(b)
copied = st1["bytes_copied"] - st0["bytes_copied"]
print(f"mode {mode_name} pool {frac:.2f}: device {dev_ms / N:.3f} ms/batch, wall {1e3 * wall / N:.3f} ms/batch, "
      f"host submit median {1e3 * np.median(host):.3f} ms max {1e3 * np.max(host):.3f} ms, "
      f"copied {copied / N / 1e6:.1f} MB/batch ({st1['loads'] - st0['loads']} slot loads) -> "
      f"{copied / (dev_ms / 1e3) / 1e9:.1f} GB/s over the device time", flush=True)
print("host submit ms per batch:", " ".join(f"{1e3 * h:.2f}" for h in host), flush=True)
# host-only cost: submit with the GPU idle between calls
hs = []
for i in range(6):
    inst, _, lens = batches[i]
    eng.synchronize()
    h0 = time.perf_counter()
    eng.infer_batch_device(inst, d_tok[i].data_ptr(), wl.seq, d_len[i].data_ptr(), int(lens.max()),
                           d_scores.data_ptr(), d_labels.data_ptr())
    hs.append(time.perf_counter() - h0)
eng.synchronize()
print("isolated host submit ms:", " ".join(f"{1e3 * h:.2f}" for h in hs), flush=True)
# copy-only probe: pinned host buffer -> device, 200 KB pieces, cudaMemcpyAsync and one big copy
piece = 200704
n = 512
hbuf = torch.empty(piece * n, dtype=torch.uint8).pin_memory()
dbuf = torch.empty(piece * n, dtype=torch.uint8, device=dev)
s2 = torch.cuda.Stream()
for big in (True, False):
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s2):
        e0.record()
        if big:
            dbuf.copy_(hbuf, non_blocking=True)
        else:
            for k in range(n):
                dbuf[k * piece:(k + 1) * piece].copy_(hbuf[k * piece:(k + 1) * piece], non_blocking=True)
        e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"H2D {'one copy' if big else f'{n} x 200 KB copies'}: {piece * n / ms / 1e6:.1f} GB/s", flush=True)
eng.close()
