# SPDX-License-Identifier: Apache-2.0
"""Pins the C restatement (oracle/hmi_oracle.c) to the reference itself.

The reference is compiled from /root/reference/proj by oracle/build_ref.sh;
these tests are skipped where neither it nor the sources exist (the committed
fixtures in tests/golden/ cover that case, see test_golden.py).
"""
import numpy as np
import pytest

import oracle
from tests.synth_tables import make_requests, make_tree

if oracle.ref() is None:  # pragma: no cover
    pytest.skip("reference library unavailable", allow_module_level=True)

SMALL = oracle.Config(64, 2, 2, 2, 128, 200, 0, 3, 11)


def _ref_tree(tables, cfg):
    t0 = tables[0]
    rt = oracle.RefTree(cfg.max_fragment, cfg.hidden_size, t0["key_len"], t0["keys"], t0["reps"])
    for t in tables[1:]:
        v = rt.add_branch(t["parent"], t["key_len"], t["keys"], t["reps"])
        assert v == t["version"]
    return rt


def _orc_tree(tables, cfg):
    ot = oracle.OracleTree(cfg.max_fragment, cfg.hidden_size)
    for t in tables:
        ot.add_table(t["version"], t["parent"], t["key_len"], t["keys"], t["reps"])
    return ot


def test_generate_model_bit_exact():
    cfg = SMALL
    m = oracle.RefModel(cfg)
    assert np.array_equal(m.higher().view(np.uint32), oracle.generate_higher(cfg).view(np.uint32))
    full = oracle.generate_model(cfg, lower=True)
    assert np.array_equal(full["higher"], m.higher())


def test_generate_adapter_and_head_bit_exact():
    cfg = SMALL
    t = oracle.RefTask(cfg, "task-7", 8, 1007, 5, 2_000_007)
    assert np.array_equal(t.adapter_f32().view(np.uint32),
                          oracle.generate_adapter(cfg, 8, 1007).view(np.uint32))
    w, b = t.head_f32()
    w2, b2 = oracle.generate_head(cfg.hidden_size, 5, 2_000_007)
    assert np.array_equal(w, w2) and np.array_equal(b, b2)


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("ngram", [2, 3, 5])
def test_retrieve_bit_exact(mode, ngram):
    cfg = oracle.Config(32, 2, 2, 2, 64, 150, mode, ngram, 3)
    tables, hot = make_tree(ngram * 10 + mode, cfg.vocab_size, cfg.hidden_size, ngram,
                            branches=((0, 30), (0, 30), (1, 20), (3, 10)))
    rt, ot = _ref_tree(tables, cfg), _orc_tree(tables, cfg)
    toks, lens = make_requests(5 + ngram, 40, hot, cfg.vocab_size, 20)
    for i in range(len(lens)):
        version = i % len(tables)
        t = toks[i, :lens[i]]
        h_ref, lev_ref = rt.retrieve(version, t, mode)
        h_orc, gather, lev_orc, srcs = ot.retrieve(version, t, mode)
        assert np.array_equal(h_ref.view(np.uint64), h_orc.view(np.uint64))
        assert np.array_equal(lev_ref, lev_orc)


def test_spec_fallback_levels():
    """SPEC.md:258-260 examples: (3,3,3), (2,2,2), (1,1,1)."""
    d, V = 8, 20
    uni = [(t,) for t in range(V)]
    keys = uni + [(1, 2, 3), (4, 5), (5, 6)]
    keys = sorted(keys)
    key_len = np.array([len(k) for k in keys], np.uint32)
    karr = np.zeros((len(keys), 3), np.uint32)
    for i, k in enumerate(keys):
        karr[i, :len(k)] = k
    reps = np.random.default_rng(0).standard_normal((int(key_len.sum()), d)).astype(np.float32)
    ot = oracle.OracleTree(3, d)
    ot.add_table(0, 0xFFFFFFFF, key_len, karr, reps)
    rt = oracle.RefTree(3, d, key_len, karr, reps)
    for toks, want in [((1, 2, 3), (3, 3, 3)), ((4, 5, 6), (2, 2, 2)), ((7, 8, 9), (1, 1, 1))]:
        # causal mode: the last position's window is the whole 3-gram
        _, _, lev, _ = ot.retrieve(0, np.array(toks), 1)
        _, rlev = rt.retrieve(0, np.array(toks), 1)
        assert lev[2, 0] == want[2] and rlev[2, 0] == want[2]
    # middle token of (4,5,6) comes from the LEFT bi-gram (leftmost rule)
    _, gather, lev, _ = ot.retrieve(0, np.array([4, 5, 6]), 1)
    row_45 = int(np.cumsum(np.r_[0, key_len])[keys.index((4, 5))])
    # position 1 of the causal window [4,5] (length 2) resolves the whole bigram (4,5)
    assert gather[1, 0] == row_45 + 1


def test_branch_shadows_root():
    d, V = 4, 10
    root_keys = sorted([(t,) for t in range(V)] + [(1, 2, 3)])
    kl = np.array([len(k) for k in root_keys], np.uint32)
    ka = np.zeros((len(root_keys), 3), np.uint32)
    for i, k in enumerate(root_keys):
        ka[i, :len(k)] = k
    reps = np.arange(int(kl.sum()) * d, dtype=np.float32).reshape(-1, d)
    ot = oracle.OracleTree(3, d)
    ot.add_table(0, 0xFFFFFFFF, kl, ka, reps)
    br = np.full((3, d), -1.0, np.float32)
    ot.add_table(1, 0, np.array([3], np.uint32), np.array([[1, 2, 3]], np.uint32), br)
    h_root, _, _, src_root = ot.retrieve(0, np.array([1, 2, 3]), 1)
    h_br, _, _, src_br = ot.retrieve(1, np.array([1, 2, 3]), 1)
    assert src_root[2, 0] == 0 and src_br[2, 0] == 1
    assert (h_br[2] == -1).all() and (h_root[2] != -1).all()


def test_forward_bit_exact_scalar():
    """Full request path vs the reference with HMI_KERNELS=scalar: bit-identical."""
    cfg = SMALL
    oracle.ref_set_kernels("scalar")
    try:
        tables, hot = make_tree(1, cfg.vocab_size, cfg.hidden_size)
        rt, ot = _ref_tree(tables, cfg), _orc_tree(tables, cfg)
        model = oracle.RefModel(cfg)
        higher = model.higher()
        n = 6
        tasks = [oracle.RefTask(cfg, f"t{i}", 8, 1000 + i, 5, 2_000_000 + i) for i in range(n)]
        toks, lens = make_requests(2, n, hot, cfg.vocab_size, 16, min_len=1)
        versions = np.arange(n) % len(tables)
        scores, labels = oracle.ref_infer(model, rt, versions, tasks, toks, lens, 5)
        for i in range(n):
            w, b = tasks[i].head_f32()
            s, lab, _ = oracle.infer_one(cfg, higher, ot, int(versions[i]), toks[i, :lens[i]],
                                         tasks[i].adapter_f32(), 8, w, b)
            assert np.array_equal(s.view(np.uint64), scores[i].view(np.uint64)), i
            assert lab == labels[i]
    finally:
        oracle.ref_set_kernels("avx2")


def test_causal_forward_bit_exact_scalar():
    cfg = oracle.Config(64, 2, 2, 2, 128, 200, 1, 3, 5)
    oracle.ref_set_kernels("scalar")
    try:
        tables, hot = make_tree(3, cfg.vocab_size, cfg.hidden_size, branches=((0, 20),))
        rt, ot = _ref_tree(tables, cfg), _orc_tree(tables, cfg)
        model = oracle.RefModel(cfg)
        tasks = [oracle.RefTask(cfg, f"t{i}", 8, 10 + i, 7, 20 + i, head_kind=2) for i in range(3)]
        toks, lens = make_requests(4, 3, hot, cfg.vocab_size, 12, min_len=2)
        versions = np.array([0, 1, 1])
        scores, labels = oracle.ref_infer(model, rt, versions, tasks, toks, lens, 7)
        for i in range(3):
            w, b = tasks[i].head_f32()
            s, lab, _ = oracle.infer_one(cfg, model.higher(), ot, int(versions[i]),
                                         toks[i, :lens[i]], tasks[i].adapter_f32(), 8, w, b,
                                         head_kind=2)
            assert np.array_equal(s, scores[i]) and lab == labels[i]
    finally:
        oracle.ref_set_kernels("avx2")


def test_padding_invariance():
    """Rows >= valid_len never influence valid rows (model.cpp:48-51): padding a request
    with zero rows (stage_compute's batch padding) leaves its head output unchanged."""
    cfg = SMALL
    higher = oracle.generate_higher(cfg)
    ad = oracle.generate_adapter(cfg, 8, 3)
    w, b = oracle.generate_head(cfg.hidden_size, 5, 4)
    h = np.random.default_rng(0).standard_normal((7, cfg.hidden_size))
    s1, l1, _, _ = oracle.higher_forward(cfg, higher, h, 7, ad, 8, w, b)
    hp = np.zeros((16, cfg.hidden_size))
    hp[:7] = h
    s2, l2, _, _ = oracle.higher_forward(cfg, higher, hp, 7, ad, 8, w, b)
    assert np.array_equal(s1, s2) and l1 == l2
