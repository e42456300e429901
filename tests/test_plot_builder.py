# SPDX-License-Identifier: Apache-2.0
"""GPU PLOT builder: build_root / derive_branch key selection
bit-exact against the reference (table.cpp:16-104), lower_stack_forward reps on the B200
against the oracle (model.cpp:96-118), and tables built on the GPU serving requests within
the logit tolerance of the reference's own tables."""
import numpy as np
import pytest

import oracle
from paper_2504_17449_b200 import plot
from paper_2504_17449_b200._native import BuildError, ConfigError, DimensionError, VocabularyError

GOLD = "tests/golden/golden_build_root.npz"


def _corpus(seed, n_seq, length, lo, hi, ragged=True):
    rng = np.random.default_rng(seed)
    out = []
    for s in range(n_seq):
        n = int(rng.integers(0, length + 1)) if ragged else length
        out.append(rng.integers(lo, hi, n).astype(np.uint32))
    return out


def _as_pairs(t):
    return [(tuple(int(x) for x in k[:l]), int(f)) for k, l, f in zip(t["keys"], t["key_len"], t["freq"])]


def test_select_matches_reference_golden():
    g = np.load(GOLD)
    root = plot.select_root(g["corpus"], 3, int(g["cfg"][5]))
    assert np.array_equal(root["key_len"], g["t0_key_len"])
    assert np.array_equal(root["keys"], g["t0_keys"])
    assert np.array_equal(root["freq"], g["t0_freq"])
    br = plot.select_branch(g["domain"], 3, 50.0)
    assert np.array_equal(br["key_len"], g["t1_key_len"])
    assert np.array_equal(br["keys"], g["t1_keys"])
    assert np.array_equal(br["freq"], g["t1_freq"])


@pytest.mark.parametrize("seed,ngram", [(1, 3), (2, 2), (3, 5), (4, 1)])
def test_select_matches_restatement(seed, ngram):
    corpus = _corpus(seed, 9, 40, 0, 25)  # ragged, including sequences shorter than ngram
    assert _as_pairs(plot.select_root(corpus, ngram, 60)) == oracle.plot_select_root(corpus, ngram, 60)
    for alpha in (0.0, 0.005, 12.345, 50.0, 99.99, 100.0):
        got = _as_pairs(plot.select_branch(corpus, ngram, alpha))
        assert got == oracle.plot_select_branch(corpus, ngram, alpha), alpha


@pytest.mark.skipif(oracle.ref() is None, reason="oracle/_ref (the compiled reference) not built")
@pytest.mark.parametrize("seed", [11, 12])
def test_select_and_lower_forward_vs_reference(seed):
    """The reference's own build_root / derive_branch: keys and frequencies equal the product's
    selection; its reps equal the C oracle's lower_stack_forward bit for bit (scalar kernels)."""
    import ctypes

    cfg = oracle.Config(128, 2, 2, 2, 256, 64, seed % 2, 3, 5 + seed)
    model = oracle.RefModel(cfg)
    corpus = _corpus(seed, 4, 14, 0, 30)
    dom = _corpus(seed + 50, 5, 14, 10, 45)
    L = oracle.ref()
    oracle.ref_set_kernels("scalar")
    try:
        lens = np.array([len(s) for s in corpus], np.uint32)
        toks = np.concatenate(corpus).astype(np.uint32)
        h = L.ref_tree_build_root(model.h, len(corpus), oracle.ptr(lens, oracle.u32p),
                                  oracle.ptr(toks, oracle.u32p))
        assert h
        rt = oracle.RefTree(3, cfg.hidden_size, None, None, None, handle=h)
        dl = np.array([len(s) for s in dom], np.uint32)
        dt = np.concatenate(dom).astype(np.uint32)
        assert L.ref_tree_derive_branch(h, model.h, len(dom), oracle.ptr(dl, oracle.u32p),
                                        oracle.ptr(dt, oracle.u32p), ctypes.c_double(37.5)) == 1
    finally:
        oracle.ref_set_kernels("avx2")
    kl0, k0, r0, f0, _ = rt.export(0)
    kl1, k1, r1, f1, _ = rt.export(1)
    root = plot.select_root(corpus, 3, cfg.vocab_size)
    br = plot.select_branch(dom, 3, 37.5)
    assert np.array_equal(root["key_len"], kl0) and np.array_equal(root["keys"], k0)
    assert np.array_equal(root["freq"], f0)
    assert np.array_equal(br["key_len"], kl1) and np.array_equal(br["keys"], k1)
    assert np.array_equal(br["freq"], f1)
    m = oracle.generate_model(cfg, lower=True)
    row = 0
    for e in range(0, len(kl0), 7):
        start = int(kl0[:e].sum())
        rep = oracle.lower_forward(cfg, m, k0[e, :kl0[e]])
        assert np.array_equal(rep.astype(np.float32), r0[start:start + kl0[e]]), e
        row += 1


def test_select_errors():
    with pytest.raises(BuildError):
        plot.select_root([], 3, 10)
    with pytest.raises(ConfigError):
        plot.select_branch([np.arange(5)], 3, 100.5)
    assert len(plot.select_branch([np.arange(2)], 3, 50.0)["key_len"]) == 0  # no 3-grams
    assert len(plot.select_branch([np.arange(9)], 3, 0.0)["key_len"]) == 0


# ---------------------------------------------------------------------------- GPU
def _rel(a, b):
    return float(np.abs(a.astype(np.float64) - b).max() / np.abs(b).max())


@pytest.mark.gpu
@pytest.mark.parametrize("mode", [0, 1])
def test_gpu_lower_forward_vs_oracle(mode):
    cfg = oracle.Config(256, 4, 2, 2, 1024, 1024, mode, 3, 7)
    from paper_2504_17449_b200 import engine as E

    mc = E.model_config(*oracle.astuple(cfg))
    b = plot.GpuPlotBuilder(mc, max_rows=256)  # several GPU passes per fragment length
    rng = np.random.default_rng(3 + mode)
    n = 400
    kl = rng.integers(1, 4, n).astype(np.uint32)
    keys = np.zeros((n, 3), np.uint32)
    for i in range(n):
        keys[i, :kl[i]] = rng.integers(0, cfg.vocab_size, kl[i])
    reps = b.forward(kl, keys)
    m = oracle.generate_model(cfg, lower=True)
    row, worst = 0, 0.0
    for i in range(n):
        ref = oracle.lower_forward(cfg, m, keys[i, :kl[i]])
        worst = max(worst, _rel(reps[row:row + kl[i]], ref))
        row += int(kl[i])
    print(f"lower stack reps (mode {mode}): max rel err {worst:.3e}")
    assert worst <= 2e-2
    with pytest.raises(DimensionError):
        b.forward(np.array([4], np.uint32), np.zeros((1, 3), np.uint32))
    with pytest.raises(VocabularyError):
        b.forward(np.array([1], np.uint32), np.array([[cfg.vocab_size, 0, 0]], np.uint32))
    b.close()


@pytest.mark.gpu
def test_gpu_built_tables_serve_within_tolerance():
    """build_root + derive_branch on the GPU over the golden corpora: keys / frequencies equal
    the reference's tables, reps within the tolerance, and an engine serving from the GPU-built
    tables reproduces the reference's logits (served from its own tables)."""
    from paper_2504_17449_b200 import engine as E
    from tests.world import logit_error

    g = np.load(GOLD)
    cfg = oracle.Config(*[int(x) for x in g["cfg"]])
    mc = E.model_config(*oracle.astuple(cfg))
    b = plot.GpuPlotBuilder(mc)
    root = b.build_root(g["corpus"])
    br = b.derive_branch(root, g["domain"], 50.0)
    for t, p in ((root, "t0"), (br, "t1")):
        assert np.array_equal(t["key_len"], g[f"{p}_key_len"])
        assert np.array_equal(t["keys"], g[f"{p}_keys"])
        assert np.array_equal(t["freq"], g[f"{p}_freq"])
        err = _rel(t["reps"], g[f"{p}_reps"].astype(np.float64))
        print(f"{p} reps max rel err {err:.3e}")
        assert err <= 2e-2
    n = len(g["lens"])
    R, LABELS = 8, 5
    eng = E.GpuEngine(mc, E.generate_higher(mc), max_batch=n, max_seq=g["tokens"].shape[1],
                      bottleneck=R, max_labels=LABELS, max_tasks=n, max_versions=8)
    eng.upload_table(0, 0xFFFFFFFF, root["key_len"], root["keys"], root["reps"])
    eng.upload_table(1, 0, br["key_len"], br["keys"], br["reps"])
    for i in range(n):
        eng.register_task(i, E.generate_adapter(mc, R, 1000 + i))
        w, bb = E.generate_head(cfg.hidden_size, LABELS, 2_000_000 + i)
        eng.register_head(i, 0, w, bb)
        eng.bind_instance(i, int(g["versions"][i]), i, i)
    res = eng.infer_batch(np.arange(n), g["tokens"], g["lens"])
    err = logit_error(res.scores, g["scores"])
    print(f"served from GPU-built tables: logit err {err:.3e}")
    assert err <= 2e-2
    assert (res.labels == g["labels"]).all()
    eng.close()
    b.close()


def test_spec_build_root_and_alpha_kats():
    """SPEC known answers: build_root over [[5, 6, 7]] holds (5), (6), (7), (5, 6),
    (6, 7), (5, 6, 7) plus every vocabulary uni-gram; (5, 6) occurs twice in
    [[5, 6, 5, 6]]; with counts {A: 5, B: 3, C: 2} alpha = 50 keeps {A}."""
    t = plot.select_root([np.array([5, 6, 7])], 3, 10)
    keys = {k for k, _ in _as_pairs(t)}
    assert {(5,), (6,), (7,), (5, 6), (6, 7), (5, 6, 7)} <= keys
    assert all((v,) in keys for v in range(10)) and len(keys) == 10 + 3
    f = dict(_as_pairs(plot.select_root([np.array([5, 6, 5, 6])], 3, 10)))
    assert f[(5, 6)] == 2 and f[(6, 5)] == 1 and f[(0,)] == 1
    # three distinct 2-grams with counts A=5, B=3, C=2 (ngram = 2 so each sequence is one 2-gram)
    A, B, C = (1, 2), (3, 4), (5, 6)
    corpus = [np.array(A)] * 5 + [np.array(B)] * 3 + [np.array(C)] * 2
    kept = [k for k, _ in _as_pairs(plot.select_branch(corpus, 2, 50.0))]
    assert kept == [A]
    kept = [k for k, _ in _as_pairs(plot.select_branch(corpus, 2, 50.01))]
    assert kept == [A, B]  # alpha monotonicity: a larger share keeps a superset
