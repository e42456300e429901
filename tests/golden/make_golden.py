# SPDX-License-Identifier: Apache-2.0
"""Generates tests/golden/*.npz from the REFERENCE itself (oracle/_ref, compiled from
/root/reference/proj/src by oracle/build_ref.sh). Run in the build container:

    python tests/golden/make_golden.py

Fixtures (all outputs computed by the reference with HMI_KERNELS=scalar, the
numeric contract of proj/src/tensor/kernels_scalar.cpp):

* golden_forward.npz — seeded synthetic PLOT tree (tests/synth_tables.py) +
  generate_model / generate_adapter_set / generate_output_head: per-request
  retrieve_sequence output (f64), resolve_window levels, head scores (f64) and
  labels of higher_stack_forward, in encoder mode.
* golden_causal.npz  — the same for causal mode with an lm_logits head.
* golden_build_root.npz — a root table built by the reference's own
  build_root (real lower_stack_forward reps over a tiny corpus) and a
  derive_branch(alpha=50) branch, plus retrieval/forward outputs over it.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402
from tests.synth_tables import make_requests, make_tree  # noqa: E402

GOLDEN_CFG = oracle.Config(128, 2, 2, 2, 256, 300, 0, 3, 17)
R, LABELS = 8, 5


def _world(cfg, tables, n_req, seed, head_kind, max_len=24):
    rt = oracle.RefTree(cfg.max_fragment, cfg.hidden_size, tables[0]["key_len"], tables[0]["keys"],
                        tables[0]["reps"])
    for t in tables[1:]:
        assert rt.add_branch(t["parent"], t["key_len"], t["keys"], t["reps"]) == t["version"]
    return rt


def _run(cfg, tables, hot, seed, head_kind, n_req=8, max_len=24, min_len=1):
    oracle.ref_set_kernels("scalar")
    rt = _world(cfg, tables, n_req, seed, head_kind)
    model = oracle.RefModel(cfg)
    toks, lens = make_requests(seed, n_req, hot, cfg.vocab_size, max_len, min_len=min_len)
    versions = (np.arange(n_req) % len(tables)).astype(np.uint32)
    tasks = [oracle.RefTask(cfg, f"task{i}", R, 1000 + i, LABELS, 2_000_000 + i, head_kind)
             for i in range(n_req)]
    scores, labels = oracle.ref_infer(model, rt, versions, tasks, toks, lens, LABELS)
    h0 = np.zeros((n_req, max_len, cfg.hidden_size))
    lev = np.zeros((n_req, max_len, cfg.max_fragment), np.uint32)
    for i in range(n_req):
        h, l = rt.retrieve(int(versions[i]), toks[i, :lens[i]], cfg.mode)
        h0[i, :lens[i]] = h
        lev[i, :lens[i]] = l
    higher = model.higher()
    oracle.ref_set_kernels("avx2")
    return dict(tokens=toks, lens=lens, versions=versions, scores=scores, labels=labels, h0=h0,
                levels=lev, higher_crc=np.array([np.frombuffer(higher.tobytes(), np.uint64).sum()],
                                                np.uint64))


def main():
    assert oracle.ref() is not None, "needs oracle/_ref (the compiled reference)"
    cfg = GOLDEN_CFG
    tables, hot = make_tree(5, cfg.vocab_size, cfg.hidden_size, 3, n_hot=16, n_bi=40, n_tri=30,
                            branches=((0, 20), (0, 20), (1, 12)))
    out = _run(cfg, tables, hot, 3, 0)
    np.savez_compressed(os.path.join(HERE, "golden_forward.npz"), cfg=np.array(oracle.astuple(cfg)),
                        table_seed=5, **out)

    ccfg = oracle.Config(128, 2, 2, 2, 256, 300, 1, 3, 19)
    tables, hot = make_tree(6, ccfg.vocab_size, ccfg.hidden_size, 3, n_hot=16, n_bi=40, n_tri=30,
                            branches=((0, 20),))
    out = _run(ccfg, tables, hot, 4, 2, min_len=2)
    np.savez_compressed(os.path.join(HERE, "golden_causal.npz"), cfg=np.array(oracle.astuple(ccfg)),
                        table_seed=6, **out)

    # real build_root / derive_branch through the reference's lower stack
    bcfg = oracle.Config(128, 2, 2, 2, 256, 96, 0, 3, 23)
    model = oracle.RefModel(bcfg)
    rng = np.random.default_rng(8)
    corpus = rng.integers(0, 40, (3, 16)).astype(np.uint32)
    L = oracle.ref()
    tree_h = L.ref_tree_build_root(model.h, 3, oracle.ptr(np.full(3, 16, np.uint32), oracle.u32p),
                                   oracle.ptr(corpus, oracle.u32p))
    assert tree_h
    rt = oracle.RefTree(3, bcfg.hidden_size, None, None, None, handle=tree_h)
    dom = rng.integers(20, 60, (4, 16)).astype(np.uint32)
    v = L.ref_tree_derive_branch(tree_h, model.h, 4, oracle.ptr(np.full(4, 16, np.uint32), oracle.u32p),
                                 oracle.ptr(dom, oracle.u32p), 50.0)
    assert v == 1
    tabs = []
    for ver in (0, 1):
        kl, keys, reps, freq, parent = rt.export(ver)
        tabs.append({"version": ver, "parent": parent, "key_len": kl, "keys": keys, "reps": reps,
                     "freq": freq})
    # serve from the float32 tables, as after PLT1 persist/load (plot_io.cpp:17-73):
    # build_root keeps full-f64 reps in memory, the served artefact is f32
    rt_built = rt
    rt = oracle.RefTree(3, bcfg.hidden_size, tabs[0]["key_len"], tabs[0]["keys"], tabs[0]["reps"],
                        tabs[0]["freq"])
    assert rt.add_branch(0, tabs[1]["key_len"], tabs[1]["keys"], tabs[1]["reps"], tabs[1]["freq"]) == 1
    fixture = {}
    for t in tabs:
        for k in ("key_len", "keys", "reps", "freq"):
            fixture[f"t{t['version']}_{k}"] = t[k]
        fixture[f"t{t['version']}_parent"] = np.array([t["parent"]], np.uint32)
    oracle.ref_set_kernels("scalar")
    toks = np.concatenate([corpus[:2, :12], dom[:2, :12]]).astype(np.uint32)
    lens = np.array([12, 7, 12, 5], np.uint32)
    versions = np.array([0, 0, 1, 1], np.uint32)
    tasks = [oracle.RefTask(bcfg, f"b{i}", R, 1000 + i, LABELS, 2_000_000 + i) for i in range(4)]
    scores, labels = oracle.ref_infer(model, rt, versions, tasks, toks, lens, LABELS)
    h0 = np.zeros((4, 12, bcfg.hidden_size))
    for i in range(4):
        h0[i, :lens[i]] = rt.retrieve(int(versions[i]), toks[i, :lens[i]], 0)[0]
    oracle.ref_set_kernels("avx2")
    np.savez_compressed(os.path.join(HERE, "golden_build_root.npz"), cfg=np.array(oracle.astuple(bcfg)),
                        corpus=corpus, domain=dom, tokens=toks, lens=lens, versions=versions,
                        scores=scores, labels=labels, h0=h0, **fixture)
    rt_built.h = None  # handle freed with the process
    print("fixtures written to", HERE)


if __name__ == "__main__":
    main()
