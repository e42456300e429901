# SPDX-License-Identifier: Apache-2.0
"""End-to-end parity of the CUDA backend against the CPU oracle.

Bar (BASELINE.json north_star): routing and gather indices bit-exact; logits
within max_i ||d_i||_inf / ||ref_i||_inf <= 2e-2; argmax agreement >= 99.9%.
The retrieval output h0 is additionally compared bit-exactly in f64.
"""
import numpy as np
import pytest

import oracle
from paper_2504_17449_b200 import engine as E
from paper_2504_17449_b200._native import RoutingError, VocabularyError
from tests.world import World, logit_error, token_tag_check

pytestmark = pytest.mark.gpu

TOL = 2e-2


@pytest.fixture(scope="module")
def c1():
    # C1 tiny hBERT: d=256, 4 heads, 2 PLOT + 2 higher layers, ffn 1024, vocab 1024, r=16
    return World(oracle.TINY, n_tasks=16, r=16, labels=8, max_batch=32)


def test_c1_parity(c1):
    inst, toks, lens = c1.requests(7, 32, 128, min_len=1)
    lens[:4] = [1, 2, 3, 128]
    c1.eng.set_debug(1)
    res = c1.eng.infer_batch(inst, toks, lens)
    ref_scores, ref_labels, _ = c1.oracle_batch(inst, toks, lens)
    err = logit_error(res.scores, ref_scores)
    agree = float((res.labels == ref_labels).mean())
    print(f"C1 logit err {err:.3e}, argmax agreement {agree:.4f}")
    assert err <= TOL
    assert agree >= 0.999

    # routing, bit-exact
    v, t, h, slots = c1.eng.debug_routing(len(inst))
    assert np.array_equal(v, c1.inst_version[inst])
    assert np.array_equal(t, inst) and np.array_equal(h, inst)
    for l in range(c1.cfg.higher_layers):
        for i, task in enumerate(inst):
            assert slots[l, i] == c1.eng.pool_slot(int(task), l) >= 0

    # gather indices and levels, bit-exact; h0 bit-exact in f64
    rows, lev = c1.eng.debug_gather(len(inst))
    S = rows.shape[1]
    h0 = c1.eng.debug_h0(len(inst), S)
    for i in range(len(inst)):
        n = int(lens[i])
        out, gather, levels, _ = c1.tree.retrieve(int(c1.inst_version[inst[i]]), toks[i, :n], 0)
        assert np.array_equal(rows[i, :n], gather.astype(np.int32)), i
        assert np.array_equal(lev[i, :n], levels.astype(np.int32)), i
        assert (rows[i, n:] == -1).all() and (lev[i, n:] == 0).all()
        assert np.array_equal(h0[i, :n].view(np.uint64), out.view(np.uint64)), i
        assert (h0[i, n:] == 0).all()
    c1.eng.set_debug(0)


def test_c1_modes_identical(c1):
    """SPEC.md:482 / acceptance #2: results identical across sync/coarse/fine."""
    inst, toks, lens = c1.requests(11, 24, 96)
    outs = []
    for mode in (E.MODE_SYNC, E.MODE_COARSE, E.MODE_FINE):
        w = World(oracle.TINY, n_tasks=16, r=16, labels=8, max_batch=32, pipeline_mode=mode)
        outs.append(w.eng.infer_batch(inst, toks, lens))
        w.eng.close()
    for o in outs[1:]:
        assert np.array_equal(o.scores, outs[0].scores)
        assert np.array_equal(o.labels, outs[0].labels)


def test_c1_permutation_and_batch_independence(c1):
    """Requests are independent: permuting a batch permutes outputs exactly, and a
    request's result does not depend on the rest of its batch (same padded length)."""
    inst, toks, lens = c1.requests(13, 20, 128)
    lens[0] = 128
    a = c1.eng.infer_batch(inst, toks, lens)
    perm = np.random.default_rng(0).permutation(20)
    perm = np.r_[0, perm[perm != 0]]  # keep a full-length request so S is unchanged
    b = c1.eng.infer_batch(inst[perm], toks[perm], lens[perm])
    assert np.array_equal(a.scores[perm], b.scores)
    single = c1.eng.infer_batch(inst[:1], toks[:1], lens[:1])
    assert np.array_equal(single.scores[0], a.scores[0])


def test_submit_wait_pipelined_matches_sync(c1):
    """hmi_gpu_submit_batch / hmi_gpu_wait_batch (up to four batches in flight) return
    exactly what the synchronous call returns; a fifth outstanding batch is refused."""
    from paper_2504_17449_b200._native import CapacityError

    reqs = [c1.requests(100 + k, 8 + 4 * k, 128) for k in range(5)]
    sync = [c1.eng.infer_batch(*r) for r in reqs]
    tickets = [c1.eng.submit_batch(*r) for r in reqs[:4]]
    with pytest.raises(CapacityError):
        c1.eng.submit_batch(*reqs[4])
    outs = [c1.eng.wait_batch(t) for t in tickets]
    t4 = c1.eng.submit_batch(*reqs[4])
    outs.append(c1.eng.wait_batch(t4))
    for a, b in zip(sync, outs):
        assert np.array_equal(a.scores, b.scores) and np.array_equal(a.labels, b.labels)


@pytest.mark.parametrize("mode", [E.MODE_COARSE, E.MODE_FINE])
def test_async_submits_pool_of_one_and_a_half_batches(c1, mode):
    """A slot pool holding 1.5 batches' working sets with three batches in flight: a load
    blocked by pinned in-flight tenants retires the oldest batch and retries. The decisions the
    blocked attempt made first (earlier tenants' loads, evictions) stand, as in the reference
    (device_pool.cpp:50-136), so their copies and slot-table deltas must still be issued —
    otherwise those tenants would route to stale slots. Scores equal the all-resident engine."""
    layer_bytes = (256 * 16 * 2 + 16 + 256) * 4
    kw = dict(n_tasks=48, r=16, labels=8, max_batch=8)
    w = World(oracle.TINY, pool_bytes=12 * 2 * layer_bytes + 100, pipeline_mode=mode, **kw)
    ref = World(oracle.TINY, **kw)
    reqs = []
    for k in range(9):
        _, toks, lens = ref.requests(300 + k, 8, 128)
        inst = (np.arange(8) + 8 * (k % 6)).astype(np.uint32)  # 8 fresh tenants per batch
        reqs.append((inst, toks, lens))
    expect = [ref.eng.infer_batch(*r) for r in reqs]
    tickets, outs = [], []
    for r in reqs:
        tickets.append(w.eng.submit_batch(*r))
        if len(tickets) == 3:
            outs.append(w.eng.wait_batch(tickets.pop(0)))
    outs += [w.eng.wait_batch(t) for t in tickets]
    for k, (a, b) in enumerate(zip(expect, outs)):
        assert np.array_equal(a.scores, b.scores), k
    st = w.eng.pool_stats()
    assert st["max_resident_bytes_seen"] <= st["capacity_bytes"]
    w.eng.synchronize()
    w.eng.close()
    ref.eng.close()


@pytest.mark.parametrize("mode", [E.MODE_SYNC, E.MODE_COARSE, E.MODE_FINE])
def test_stage_trace_invariants(mode):
    """StageTrace: end >= start; intervals of one worker never
    overlap; a layer's compute starts after that layer's adapter prefetch ends (fine), or after
    all of the batch's prefetches (sync / coarse); sync also waits for the previous batch."""
    layer_bytes = (256 * 16 * 2 + 16 + 256) * 4
    w = World(oracle.TINY, n_tasks=16, r=16, labels=8, max_batch=8,
              pool_bytes=6 * 2 * layer_bytes + 100, pipeline_mode=mode)
    w.eng.trace(True)
    for k in range(4):
        inst, toks, lens = w.requests(60 + k, 6, 128)
        w.eng.infer_batch((inst + 5 * k) % 16, toks, lens)
    recs = w.eng.stage_trace()
    w.eng.trace(False)
    w.eng.close()
    assert len(recs) == 4 * (2 + 2 * 2 + 1)  # per batch: host, retrieve, 2 x (prefetch, compute), head
    eps = 1e-3
    for r in recs:
        assert r["end_ms"] >= r["start_ms"] - eps, r
    for wk in ("cpu", "io", "compute"):
        iv = sorted((r["start_ms"], r["end_ms"]) for r in recs if r["worker"] == wk)
        for (a0, a1), (b0, b1) in zip(iv, iv[1:]):
            assert b0 >= a1 - eps, (wk, (a0, a1), (b0, b1))
    for b in {r["batch"] for r in recs}:
        pre = {r["layer"]: r for r in recs if r["batch"] == b and r["stage"] == "prefetch"}
        comp = {r["layer"]: r for r in recs if r["batch"] == b and r["stage"] == "compute"}
        ret = [r for r in recs if r["batch"] == b and r["stage"] == "retrieve"][0]
        for l, c in comp.items():
            assert c["start_ms"] >= pre[l]["end_ms"] - eps
        if mode != E.MODE_FINE:
            assert ret["start_ms"] >= max(p["end_ms"] for p in pre.values()) - eps


def test_zero_adapter_is_identity():
    """SPEC S:124 / S:169: an adapter whose parameters are all zero is the identity, so a
    request of that tenant equals the reference's layer_forward without an adapter."""
    w = World(oracle.TINY, n_tasks=4, r=16, labels=8, max_batch=8)
    zero = np.zeros_like(w.adapters[2])
    w.eng.replace_task(2, zero)
    inst, toks, lens = w.requests(71, 8, 128, min_len=1)
    inst[:] = 2
    res = w.eng.infer_batch(inst, toks, lens)
    ref = []
    for i in range(len(inst)):
        hw, hb = w.heads[2]
        ref.append(oracle.infer_one(w.cfg, w.higher, w.tree, int(w.inst_version[2]), toks[i, :lens[i]],
                                    None, w.r, hw, hb)[0])
    ref = np.stack(ref)
    assert logit_error(res.scores, ref) <= TOL
    assert (res.labels == ref.argmax(axis=1)).mean() >= 0.999
    w.eng.close()


def test_c1_swap_small_pool_bit_identical(c1):
    """A pool holding only 3 tasks forces evictions and reloads every batch; outputs
    are bit-identical to the all-resident run and the trace obeys the LRU law."""
    layer_bytes = (256 * 16 * 2 + 16 + 256) * 4
    w = World(oracle.TINY, n_tasks=16, r=16, labels=8, max_batch=32,
              pool_bytes=3 * 2 * layer_bytes + 100, pipeline_mode=E.MODE_FINE)
    inst, toks, lens = c1.requests(17, 3, 64)
    inst[:] = [0, 5, 9]
    outs = []
    for k in range(4):
        i2 = (inst + 3 * k) % 16
        r = w.eng.infer_batch(i2, toks, lens, want_trace=True)
        ref = c1.eng.infer_batch(i2, toks, lens)
        assert np.array_equal(r.scores, ref.scores)
        assert any(not t["hit"] for t in r.trace)
        outs.append(r)
    st = w.eng.pool_stats()
    assert st["max_resident_bytes_seen"] <= st["capacity_bytes"]
    assert st["loads"] > 0
    w.eng.close()


BASE_SMALL = dict(n_tasks=4, r=64, labels=8, max_batch=4, branches=tuple((0, 60) for _ in range(2)),
                  n_hot=64, n_bi=400, n_tri=400)


def test_grouped_adapter_gemms_wide_bottleneck():
    """Bottleneck r = 96 (> 64, padded to 128): the adapter runs as the O projection followed by
    the two tenant-grouped tcgen05 GEMMs (folded down + ReLU, then up + skip + LN2-residual + row
    statistics) instead of the O projection's tenant K blocks; parity against the oracle."""
    w = World(oracle.TINY, n_tasks=8, r=96, labels=8, max_batch=16)
    inst, toks, lens = w.requests(29, 16, 128)
    res = w.eng.infer_batch(inst, toks, lens)
    ref_scores, ref_labels, _ = w.oracle_batch(inst, toks, lens)
    assert logit_error(res.scores, ref_scores) <= TOL
    assert (res.labels == ref_labels).mean() >= 0.999
    w.eng.close()


@pytest.mark.parametrize("causal", [0, 1])
def test_attention_tc_parity(causal):
    """tcgen05 attention (padded length 128), encoder and causal, against the oracle."""
    cfg = oracle.Config(256, 4, 2, 2, 1024, 1024, causal, 3, 31)
    kind = E.HEAD_LM if causal else E.HEAD_CLS
    w = World(cfg, n_tasks=8, r=16, labels=8, max_batch=16, head_kind=kind)
    inst, toks, lens = w.requests(37, 16, 128, min_len=1)
    tc = w.eng.infer_batch(inst, toks, lens)
    w.eng.close()
    ref_scores, ref_labels, _ = w.oracle_batch(inst, toks, lens)
    assert logit_error(tc.scores, ref_scores) <= TOL
    assert (tc.labels == ref_labels).mean() >= 0.999


def test_routing_and_vocab_errors(c1):
    inst, toks, lens = c1.requests(3, 2, 16)
    bad = inst.copy()
    bad[1] = 999
    with pytest.raises(RoutingError):
        c1.eng.infer_batch(bad, toks, lens)
    t2 = toks.copy()
    t2[0, 0] = c1.cfg.vocab_size
    with pytest.raises(VocabularyError):
        c1.eng.infer_batch(inst, t2, lens)
    # the engine is still usable afterwards
    c1.eng.infer_batch(inst, toks, lens)


@pytest.mark.parametrize("mode", [0, 1])
def test_long_requests_s256(mode):
    """Padded length 256 (two 128-row tiles per request) takes the general attention
    kernel (online softmax over 64-key blocks) and multi-tile adapter routing."""
    cfg = oracle.Config(256, 4, 2, 2, 1024, 1024, mode, 3, 13)
    w = World(cfg, n_tasks=4, r=16, labels=8, max_batch=6, max_seq=256,
              head_kind=E.HEAD_LM if mode else E.HEAD_CLS)
    inst, toks, lens = w.requests(29, 6, 240, min_len=130)
    res = w.eng.infer_batch(inst, toks, lens)
    ref_scores, ref_labels, _ = w.oracle_batch(inst, toks, lens)
    assert logit_error(res.scores, ref_scores) <= TOL
    assert (res.labels == ref_labels).mean() >= 0.999
    w.eng.close()


@pytest.mark.parametrize("mode", [0, 1])
def test_max_length_s512_ragged(mode):
    """Maximum padded length 512 (four row tiles per request) with ragged lengths down to a
    single token in one batch: general attention path, per-tile adapter routing, causal and
    encoder, token_tag head (every position checked)."""
    cfg = oracle.Config(128, 2, 2, 2, 256, 600, mode, 3, 17)
    w = World(cfg, n_tasks=5, r=8, labels=6, max_batch=5, max_seq=512, head_kind=E.HEAD_TAG)
    inst, toks, lens = w.requests(31, 5, 512, min_len=1)
    lens[:3] = [512, 1, 385]
    w.eng.set_debug(2)
    res = w.eng.infer_batch(inst, toks, lens, want_tags=True)
    hidden = w.eng.debug_hidden(len(inst), 512)
    agree, n, decisive, ties = token_tag_check(w, inst, toks, lens, res.tags, hidden)
    print(f"s512 token_tag: {n} tokens, agreement {agree:.4f}, near-ties {len(ties)}")
    assert not decisive, decisive  # every disagreement is a near-tie within the row's error
    assert agree >= 0.99
    for i in range(len(lens)):
        assert (res.tags[i, lens[i]:] == -1).all()
    w.eng.close()


def test_token_tag_head():
    """token_tag (model.cpp:158-163): every valid row's argmax; each disagreement with the
    oracle must be a near-tie within that row's measured score error."""
    w = World(oracle.TINY, n_tasks=4, r=16, labels=5, head_kind=E.HEAD_TAG, max_batch=64)
    inst, toks, lens = w.requests(5, 64, 128, min_len=3)
    w.eng.set_debug(2)
    res = w.eng.infer_batch(inst, toks, lens, want_tags=True)
    hidden = w.eng.debug_hidden(len(inst), 128)  # padded length of the batch
    agree, n, decisive, ties = token_tag_check(w, inst, toks, lens, res.tags, hidden)
    print(f"token_tag: {n} tokens, agreement {agree:.4f}, near-ties {len(ties)}")
    assert n > 3000
    assert not decisive, decisive
    assert agree >= 0.999
    assert (res.labels == -1).all()
    w.eng.close()


def test_causal_lm_head():
    """hGPT-style: causal retrieval + causal attention, lm head on row valid_len-1."""
    cfg = oracle.Config(256, 4, 2, 2, 1024, 1024, 1, 3, 9)
    w = World(cfg, n_tasks=6, r=16, labels=64, head_kind=E.HEAD_LM, max_batch=8)
    inst, toks, lens = w.requests(21, 8, 100, min_len=2)
    res = w.eng.infer_batch(inst, toks, lens)
    ref_scores, ref_labels, _ = w.oracle_batch(inst, toks, lens)
    assert logit_error(res.scores, ref_scores) <= TOL
    assert (res.labels == ref_labels).mean() >= 0.999
    w.eng.close()


def test_bf16_operands_close():
    """bf16 operands run through the same kernels (reported alongside fp16)."""
    w = World(oracle.TINY, n_tasks=4, r=16, labels=8, max_batch=8, precision=1)
    inst, toks, lens = w.requests(31, 8, 128)
    res = w.eng.infer_batch(inst, toks, lens)
    ref_scores, _, _ = w.oracle_batch(inst, toks, lens)
    assert logit_error(res.scores, ref_scores) <= 0.1
    w.eng.close()


@pytest.mark.parametrize("n_req", [24])
def test_base_parity(n_req):
    """C2 shapes (hBERT-base: d=768, 12 heads, 6 higher layers, ffn 3072, r=64, 8 labels)."""
    w = World(oracle.BASE, n_tasks=12, r=64, labels=8, max_batch=n_req,
              branches=tuple((0, 60) for _ in range(8)), n_hot=64, n_bi=400, n_tri=400)
    inst, toks, lens = w.requests(41, n_req, 128, min_len=100)
    res = w.eng.infer_batch(inst, toks, lens)
    ref_scores, ref_labels, _ = w.oracle_batch(inst, toks, lens, threads=32)
    err = logit_error(res.scores, ref_scores)
    print(f"C2 logit err {err:.3e}, argmax agreement {(res.labels == ref_labels).mean():.4f}")
    assert err <= TOL
    assert (res.labels == ref_labels).mean() >= 0.999
    w.eng.close()


def test_full_size_batch_composition_invariance():
    """BASELINE's full C2 batch (256 requests x 128 tokens, hBERT-base, r = 64) against a
    size-independent property: each request's scores do not depend on the batch it rides in.
    The full batch, its two halves in swapped order, and a reversed permutation give the same
    scores bit for bit (rows are independent through every kernel; the GEMM tile order, the
    wave-tail split and the pipelined copies must not leak across requests)."""
    w = World(oracle.BASE, n_tasks=64, r=64, labels=8, max_batch=256,
              branches=tuple((0, 60) for _ in range(8)), n_hot=64, n_bi=400, n_tri=400)
    inst, toks, lens = w.requests(71, 256, 128, min_len=1)
    full = w.eng.infer_batch(inst, toks, lens)
    lo = w.eng.infer_batch(inst[128:], toks[128:], lens[128:])
    hi = w.eng.infer_batch(inst[:128], toks[:128], lens[:128])
    assert np.array_equal(np.concatenate([hi.scores, lo.scores]), full.scores)
    perm = np.arange(256)[::-1]
    rev = w.eng.infer_batch(inst[perm], toks[perm], lens[perm])
    assert np.array_equal(rev.scores[perm], full.scores)
    assert np.array_equal(rev.labels[perm], full.labels)
    # and a spot check of eight of them against the oracle
    pick = np.arange(0, 256, 32)
    ref, _, _ = w.oracle_batch(inst[pick], toks[pick], lens[pick], threads=8)
    assert logit_error(full.scores[pick], ref) <= TOL
    w.eng.close()


@pytest.mark.parametrize("mode", [E.MODE_SYNC, E.MODE_FINE])
def test_full_size_swapping_is_invisible(mode):
    """C2 shapes with a slot pool holding 20 of 64 tenants: adapters stream in and out
    between (sync) or inside (fine, per layer) batches, and every score equals the all-resident
    engine's bit for bit."""
    kw = dict(n_tasks=64, r=64, labels=8, max_batch=256, branches=tuple((0, 60) for _ in range(8)),
              n_hot=64, n_bi=400, n_tri=400)
    ref = World(oracle.BASE, **kw)
    layer_bytes = (768 * 64 * 2 + 64 + 768) * 4
    small = World(oracle.BASE, pool_bytes=20 * oracle.BASE.higher_layers * layer_bytes,
                  pipeline_mode=mode, **kw)
    for k in range(8):  # each batch: 16 tenants (its working set), the sets rotating over all 64
        inst, toks, lens = ref.requests(81 + k, 96, 128, min_len=1)
        inst = ((np.arange(96) % 16) + 16 * (k % 4) + (k // 4) * 8) % 64
        a = ref.eng.infer_batch(inst.astype(np.uint32), toks, lens)
        b = small.eng.infer_batch(inst.astype(np.uint32), toks, lens)
        assert np.array_equal(a.scores, b.scores), k
    assert small.eng.pool_stats()["bytes_copied"] > ref.eng.pool_stats()["bytes_copied"]  # re-loads
    # whole-task misses land in one block of consecutive slots: at most one transfer per missed
    # tenant, not one per (tenant, layer) (tenants registered and placed side by side share one)
    loads = small.eng.pool_stats()["loads"]
    transfers = E.engine_counters(small.eng)["adapter_copies"]
    L = oracle.BASE.higher_layers
    print(f"{loads} (tenant, layer) loads in {transfers} transfers")
    assert 1 <= transfers <= -(-loads // L)
    ref.eng.close()
    small.eng.close()


def test_large_parity_three_level_tree():
    """C5 shapes (hBERT-large: d=1024, 16 heads, 12 higher layers, ffn 4096, r=64): the folded
    adapter and the O projection's tenant K blocks at d=1024 (16 row-statistics partials), a
    3-level domain tree."""
    w = World(oracle.LARGE, n_tasks=6, r=64, labels=8, max_batch=6,
              branches=((0, 60), (0, 60), (1, 40), (2, 40)), n_hot=64, n_bi=300, n_tri=300)
    inst, toks, lens = w.requests(43, 6, 128, min_len=90)
    res = w.eng.infer_batch(inst, toks, lens)
    ref_scores, ref_labels, _ = w.oracle_batch(inst, toks, lens, threads=32)
    err = logit_error(res.scores, ref_scores)
    print(f"C5 logit err {err:.3e}, argmax agreement {(res.labels == ref_labels).mean():.4f}")
    assert err <= TOL
    assert (res.labels == ref_labels).mean() >= 0.999
    w.eng.close()


@pytest.fixture(scope="module")
def gpt():
    """hGPT-style tiny causal model, one vocabulary-wide lm head (1024 > max_labels) shared
    by every instance, KV cache for 12 generated tokens."""
    cfg = oracle.Config(256, 4, 2, 2, 1024, 1024, 1, 3, 11)
    w = World(cfg, n_tasks=8, r=16, labels=cfg.vocab_size, head_kind=E.HEAD_LM, max_batch=16,
              shared_head=True, max_new_tokens=12, max_labels=8)
    yield w
    w.eng.close()


def test_wide_lm_head_infer_batch(gpt):
    """The wide lm head through infer_batch: label = argmax over the vocabulary,
    scores[:, 0] = its logit (tcgen05 logits GEMM + f64 rescoring of the top-8)."""
    inst, toks, lens = gpt.requests(51, 16, 120, min_len=1)
    res = gpt.eng.infer_batch(inst, toks, lens)
    ref_scores, ref_labels, _ = gpt.oracle_batch(inst, toks, lens)
    assert (res.labels == ref_labels).mean() >= 0.999
    top = ref_scores[np.arange(len(inst)), ref_labels]
    rel = np.abs(res.scores[:, 0] - top) / np.abs(ref_scores).max(axis=1)
    assert rel.max() <= TOL
    assert (res.scores[:, 1:8] == 0).all()


def test_generate_teacher_forced(gpt):
    """Greedy generation with the KV cache: every generated token is checked against
    the oracle's full causal forward over prompt + the tokens generated before it
    (teacher forcing), so one near-tie cannot cascade through the comparison."""
    n, n_new = 12, 12
    inst, toks, lens = gpt.requests(53, n, 116, min_len=2)
    lens[:3] = [2, 3, 116]
    gen, logit = gpt.eng.generate(inst, toks, lens, n_new)
    assert ((gen >= 0) & (gen < gpt.cfg.vocab_size)).all()
    # the first token is what infer_batch predicts for the prompt
    res = gpt.eng.infer_batch(inst, toks, lens)
    assert np.array_equal(gen[:, 0], res.labels)
    seqs, meta = [], []
    for i in range(n):
        for k in range(n_new):
            seq = np.concatenate([toks[i, :lens[i]], gen[i, :k].astype(np.uint32)])
            seqs.append(seq)
            meta.append((i, k))
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(16) as ex:
        out = list(ex.map(lambda s: gpt.oracle_one(int(inst[meta[s][0]]), seqs[s], len(seqs[s])),
                          range(len(seqs))))
    agree, worst_gap, worst_err = 0, 0.0, 0.0
    for (i, k), (scores, label, _) in zip(meta, out):
        scale = np.abs(scores).max()
        g = int(gen[i, k])
        agree += int(g == label)
        worst_gap = max(worst_gap, (scores[label] - scores[g]) / scale)   # 0 when equal
        worst_err = max(worst_err, abs(float(logit[i, k]) - scores[g]) / scale)
    rate = agree / len(meta)
    print(f"generate: argmax agreement {rate:.4f}, worst near-tie gap {worst_gap:.2e}, "
          f"worst logit err {worst_err:.2e}")
    assert worst_err <= TOL
    assert worst_gap <= TOL          # any disagreement is a near tie within tolerance
    assert rate >= 0.97


def test_generate_graph_replay_matches_eager():
    """The decode step replayed from a captured CUDA graph produces exactly the tokens and
    logits of eager launches, across batch shapes (one graph each), repeated calls, and a
    table upload between calls (the graph is recaptured against the new retrieval state)."""
    cfg = oracle.Config(256, 4, 2, 2, 1024, 1024, 1, 3, 11)
    outs = {}
    for mode in ("1", "0"):
        w = World(cfg, n_tasks=8, r=16, labels=cfg.vocab_size, head_kind=E.HEAD_LM, max_batch=16,
                  shared_head=True, max_new_tokens=12, max_labels=8)
        w.eng.set_debug(0 if mode == "1" else 4)  # bit 2: eager decode launches
        res = []
        for seed, n, n_new in ((61, 16, 12), (62, 5, 7), (61, 16, 12)):
            inst, toks, lens = w.requests(seed, n, 100, min_len=2)
            res.append(w.eng.generate(inst, toks, lens, n_new))
        t = w.tables[-1]
        w.eng.upload_table(len(w.tables) + 1, t["version"], t["key_len"], t["keys"], t["reps"])
        inst, toks, lens = w.requests(63, 16, 100, min_len=2)
        res.append(w.eng.generate(inst, toks, lens, 12))
        outs[mode] = res
        w.eng.close()
    for (g1, l1), (g0, l0) in zip(outs["1"], outs["0"]):
        assert np.array_equal(g1, g0)
        assert np.array_equal(l1.view(np.uint32), l0.view(np.uint32))
    assert np.array_equal(outs["1"][0][0], outs["1"][2][0])  # replay is repeatable


def test_generate_after_head_arena_growth(gpt):
    """Registering another wide head reallocates the head arena (and possibly the logits
    buffer) that a captured decode graph reads by address: the graphs are dropped and
    recaptured, so generation after the registration returns what it returned before."""
    inst, toks, lens = gpt.requests(58, 16, 100, min_len=2)
    g1, l1 = gpt.eng.generate(inst, toks, lens, 12)
    w, b = E.generate_head(gpt.cfg.hidden_size, gpt.cfg.vocab_size, 3_000_000)
    gpt.eng.register_head(1, E.HEAD_LM, w, b)
    g2, l2 = gpt.eng.generate(inst, toks, lens, 12)
    assert np.array_equal(g1, g2)
    assert np.array_equal(l1.view(np.uint32), l2.view(np.uint32))


def test_generate_errors(gpt):
    inst, toks, lens = gpt.requests(55, 4, 40)
    from paper_2504_17449_b200._native import ConfigError
    with pytest.raises(ConfigError):
        gpt.eng.generate(inst, toks, lens, 13)  # > max_new_tokens


def test_generate_gpt2_small_shapes():
    """C3 shapes: hGPT-2 small (d=768, 12 heads, 6 higher layers, ffn 3072, r=64) with the
    50,257-token lm head shared by every tenant; teacher-forced against the oracle."""
    w = World(oracle.GPT2S, n_tasks=6, r=64, labels=oracle.GPT2S.vocab_size,
              head_kind=E.HEAD_LM, max_batch=6, shared_head=True, max_new_tokens=3,
              max_labels=8, branches=tuple((0, 60) for _ in range(4)), n_hot=64, n_bi=400,
              n_tri=400)
    inst, toks, lens = w.requests(57, 6, 128, min_len=100)
    gen, logit = w.eng.generate(inst, toks, lens, 3)
    from concurrent.futures import ThreadPoolExecutor
    jobs = [(i, k) for i in range(6) for k in range(3)]

    def run(j):
        i, k = j
        seq = np.concatenate([toks[i, :lens[i]], gen[i, :k].astype(np.uint32)])
        return w.oracle_one(int(inst[i]), seq, len(seq))

    with ThreadPoolExecutor(32) as ex:
        out = list(ex.map(run, jobs))
    agree = 0
    for (i, k), (scores, label, _) in zip(jobs, out):
        scale = np.abs(scores).max()
        g = int(gen[i, k])
        agree += int(g == label)
        assert (scores[label] - scores[g]) / scale <= TOL
        assert abs(float(logit[i, k]) - scores[g]) / scale <= TOL
    print(f"C3 generate argmax agreement {agree / len(jobs):.4f}")
    assert agree / len(jobs) >= 0.94
    w.eng.close()
