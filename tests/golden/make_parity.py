# SPDX-License-Identifier: Apache-2.0
"""Generates the at-scale parity fixtures tests/golden/parity_{c2,c5}.npz from the
REFERENCE itself (oracle/_ref: retrieve_sequence + higher_stack_forward per request,
compiled from /root/reference/proj/src by oracle/build_ref.sh, HMI_KERNELS=avx2).

    python tests/golden/make_parity.py [c2|c5 ...]

The worlds are BASELINE.json's own configurations, exactly as bench.py builds them
(paper_2504_17449_b200/workload.py, seeded): C2 = hBERT-base, 1,000 tenants, root + 8
domain branches over the 30,522-token vocabulary; C5 = hBERT-large, 10,000 tenants,
root -> 8 domains -> 2 sub-domains each. Requests are world.requests(seed, n): tenants
uniform over all tenants, 95% domain-corpus windows, 5% uniform vocabulary.

Stored per request: tenant / instance id, the reference's f64 head scores and first-max
label, and its top-2 margin (for reading argmax disagreements). The GPU test
(tests/test_parity_scale.py) regenerates the same requests and checks `inst` first, so a
drifted workload cannot pass against stale fixtures; it also re-runs a subset through the
C oracle live on the GPU box.
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402
from paper_2504_17449_b200.workload import CONFIGS, World  # noqa: E402

PARITY = {  # config -> (request seed, number of requests)
    "c2": (424242, 1024),
    "c5": (525252, 256),
}


def make(name: str) -> None:
    wl = CONFIGS[name]
    seed, n = PARITY[name]
    t0 = time.time()
    world = World(wl)
    inst, toks, lens = world.requests(seed, n)
    cfg = oracle.Config(wl.hidden_size, wl.heads, wl.lower_layers, wl.higher_layers, wl.ffn_size,
                        wl.vocab_size, wl.mode, wl.max_fragment, wl.model_seed)
    oracle.ref_set_kernels("avx2")
    model = oracle.RefModel(cfg)
    t = world.tables[0]
    tree = oracle.RefTree(wl.max_fragment, wl.hidden_size, t["key_len"], t["keys"], t["reps"])
    for t in world.tables[1:]:
        assert tree.add_branch(t["parent"], t["key_len"], t["keys"], t["reps"]) == t["version"]
    tasks = {int(k): oracle.RefTask(cfg, f"task{int(k)}", wl.r, 1000 + int(k), wl.labels,
                                    2_000_000 + int(k), wl.head_kind) for k in set(inst.tolist())}
    versions = np.array([world.tenant_version(int(k)) for k in inst], np.uint32)
    print(f"{name}: world ready in {time.time() - t0:.1f} s; {n} requests, "
          f"{len(tasks)} tenants", flush=True)
    t0 = time.time()
    scores, labels = oracle.ref_infer(model, tree, versions, [tasks[int(k)] for k in inst], toks,
                                      lens, wl.labels, threads=os.cpu_count() or 1)
    srt = np.sort(scores, axis=1)
    margin = (srt[:, -1] - srt[:, -2]) / np.abs(scores).max(axis=1)
    print(f"{name}: reference forward {time.time() - t0:.1f} s", flush=True)
    np.savez_compressed(os.path.join(HERE, f"parity_{name}.npz"), seed=seed, inst=inst,
                        versions=versions, scores=scores, labels=labels, margin=margin,
                        kernels=np.array(oracle.ref().ref_active_kernels().decode()))


if __name__ == "__main__":
    for name in sys.argv[1:] or list(PARITY):
        make(name)
