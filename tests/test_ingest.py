# SPDX-License-Identifier: Apache-2.0
"""Artefact ingest: PLT1 / ADP1 / HMI1 files written by the reference's
own writers read back bit-exactly into the C ABI's f32 layouts; PLT1 files written here load in
the reference's plot::load; corrupted files fail with FormatError exactly where the reference's
readers do."""
import ctypes
import os

import numpy as np
import pytest

import oracle
from paper_2504_17449_b200 import plot
from paper_2504_17449_b200._native import FormatError

GOLD = "tests/golden/golden_build_root.npz"
needs_ref = pytest.mark.skipif(oracle.ref() is None, reason="oracle/_ref not built")


def _ref_plt1(path):
    L = oracle.ref()
    hdr = np.zeros(6, np.uint32)
    rc = L.ref_plt1_load(path.encode(), oracle.ptr(hdr, oracle.u32p), None, None, None, None)
    if rc != 0:
        return rc, None
    n, ngram, d = int(hdr[4]), int(hdr[2]), int(hdr[3])
    kl = np.empty(n, np.uint32)
    assert L.ref_plt1_load(path.encode(), oracle.ptr(hdr, oracle.u32p), oracle.ptr(kl, oracle.u32p),
                           None, None, None) == 0
    keys = np.empty((n, ngram), np.uint32)
    reps = np.empty((int(kl.sum()), d), np.float32)
    freq = np.empty(n, np.uint64)
    assert L.ref_plt1_load(path.encode(), oracle.ptr(hdr, oracle.u32p), oracle.ptr(kl, oracle.u32p),
                           oracle.ptr(keys, oracle.u32p), oracle.ptr(reps, oracle.f32p),
                           oracle.ptr(freq, oracle.u64p)) == 0
    return 0, {"hdr": hdr, "key_len": kl, "keys": keys, "reps": reps, "freq": freq}


def _golden_table():
    g = np.load(GOLD)
    return {"key_len": g["t1_key_len"], "keys": g["t1_keys"], "freq": g["t1_freq"], "reps": g["t1_reps"]}


def test_plt1_round_trip(tmp_path):
    t = _golden_table()
    p = str(tmp_path / "branch.plt1")
    plot.save_plt1(t, p, 1, 0, "dom", 5000)
    u, v, par, a = plot.load_plt1(p)
    assert (v, par, a) == (1, 0, 5000)
    for k in t:
        assert np.array_equal(u[k], t[k]), k


@needs_ref
def test_plt1_interchange_with_reference(tmp_path):
    """Reference persist -> our loader, and our writer -> reference plot::load, bit-exact."""
    g = np.load(GOLD)
    rt = oracle.RefTree(3, int(g["cfg"][0]), g["t0_key_len"], g["t0_keys"], g["t0_reps"], g["t0_freq"])
    v = rt.add_branch(0, g["t1_key_len"], g["t1_keys"], g["t1_reps"], g["t1_freq"])
    p = str(tmp_path / "ref.plt1")
    assert oracle.ref().ref_plot_persist(rt.h, v, p.encode()) == 0
    u, ver, par, _ = plot.load_plt1(p)
    assert (ver, par) == (v, 0)
    for k in ("key_len", "keys", "freq", "reps"):
        assert np.array_equal(u[k], g[f"t1_{k}"]), k
    q = str(tmp_path / "ours.plt1")
    plot.save_plt1(u, q, ver, par, "x", 1234)
    rc, r = _ref_plt1(q)
    assert rc == 0
    assert list(r["hdr"]) == [ver, par, 3, int(g["cfg"][0]), len(u["key_len"]), 1234]
    for k in ("key_len", "keys", "freq", "reps"):
        assert np.array_equal(r[k], u[k]), k


@needs_ref
def test_adp1_and_hmi1_from_reference_writers(tmp_path):
    cfg = oracle.Config(128, 2, 2, 2, 256, 96, 0, 3, 23)
    task = oracle.RefTask(cfg, "tenant-7", 8, 1007, 5, 2_000_007)
    p = str(tmp_path / "t7.adp1")
    assert oracle.ref().ref_adapter_save(task.adapter, p.encode()) == 0
    name, body = plot.load_adp1(p)
    assert name == "tenant-7"
    assert np.array_equal(body, task.adapter_f32())
    assert np.array_equal(body, oracle.generate_adapter(cfg, 8, 1007))
    model = oracle.RefModel(cfg)
    q = str(tmp_path / "m.hmi1")
    assert oracle.ref().ref_model_save(model.h, q.encode()) == 0
    mc, tok, pos, low, hi = plot.load_hmi1(q)
    assert tuple(getattr(mc, f) for f, _ in mc._fields_) == oracle.astuple(cfg)
    m = oracle.generate_model(cfg, lower=True)
    assert np.array_equal(tok, m["token_embedding"]) and np.array_equal(pos, m["position_embedding"])
    assert np.array_equal(low, m["lower"]) and np.array_equal(hi, model.higher())


def _corrupt(src, dst, fn):
    b = bytearray(open(src, "rb").read())
    b = fn(b)
    open(dst, "wb").write(bytes(b))


@needs_ref
@pytest.mark.parametrize("case", ["magic", "truncated", "trailing", "zero_freq", "key_len0",
                                  "key_len_big", "duplicate", "zero_ngram"])
def test_plt1_format_errors_match_reference(tmp_path, case):
    t = _golden_table()
    good = str(tmp_path / "good.plt1")
    plot.save_plt1(t, good, 1, 0, "", 0)
    d = t["reps"].shape[1]
    hdr = 4 + 4 + 4 + 4 + 0 + 4 + 4 + 4 + 4     # magic, version, parent, label(len 0), ngram, d, n, alpha
    e0 = hdr                                    # first entry: key_len u32, key, freq u64, reps
    k0 = int(t["key_len"][0])
    e1 = e0 + 4 + 4 * k0 + 8 + 4 * k0 * d

    def edit(b):
        if case == "magic":
            b[0:4] = b"PLT2"
        elif case == "truncated":
            b = b[:-7]
        elif case == "trailing":
            b += b"\0"
        elif case == "zero_freq":
            b[e0 + 4 + 4 * k0:e0 + 12 + 4 * k0] = (0).to_bytes(8, "little")
        elif case == "key_len0":
            b[e0:e0 + 4] = (0).to_bytes(4, "little")
        elif case == "key_len_big":
            b[e0:e0 + 4] = (9).to_bytes(4, "little")
        elif case == "duplicate":  # entry 1 := entry 0 (same key)
            k1 = int(t["key_len"][1])
            assert k1 == k0
            b[e1:e1 + 4 + 4 * k0] = b[e0:e0 + 4 + 4 * k0]
        elif case == "zero_ngram":
            b[16:20] = (0).to_bytes(4, "little")
        return b

    bad = str(tmp_path / f"{case}.plt1")
    _corrupt(good, bad, edit)
    rc, _ = _ref_plt1(bad)
    assert rc == 9, (case, rc)  # the reference raises FormatError
    with pytest.raises(FormatError):
        plot.load_plt1(bad)


@needs_ref
@pytest.mark.parametrize("case", ["magic", "truncated", "trailing", "rank_ge_d"])
def test_adp1_hmi1_format_errors_match_reference(tmp_path, case):
    cfg = oracle.Config(128, 2, 2, 2, 256, 96, 0, 3, 23)
    task = oracle.RefTask(cfg, "t", 8, 1, 5, 2)
    good = str(tmp_path / "good.adp1")
    assert oracle.ref().ref_adapter_save(task.adapter, good.encode()) == 0
    rank_at = 4 + 4 + 1 + 4 + 4  # magic, str len, "t", layers, d

    def edit(b):
        if case == "magic":
            b[0:4] = b"ADP0"
        elif case == "truncated":
            b = b[:-3]
        elif case == "trailing":
            b += b"\0\0\0\0"
        elif case == "rank_ge_d":
            b[rank_at:rank_at + 4] = (128).to_bytes(4, "little")
        return b

    bad = str(tmp_path / f"{case}.adp1")
    _corrupt(good, bad, edit)
    assert oracle.ref().ref_adp1_check(bad.encode()) == 9
    with pytest.raises(FormatError):
        plot.load_adp1(bad)
    if case in ("magic", "truncated", "trailing"):
        model = oracle.RefModel(cfg)
        q = str(tmp_path / "m.hmi1")
        assert oracle.ref().ref_model_save(model.h, q.encode()) == 0
        qb = str(tmp_path / f"{case}.hmi1")
        _corrupt(q, qb, lambda b: (b.__setitem__(slice(0, 4), b"HMI0") or b) if case == "magic" else edit(b))
        assert oracle.ref().ref_hmi1_check(qb.encode()) == 9
        with pytest.raises(FormatError):
            plot.load_hmi1(qb)


@pytest.mark.gpu
def test_gpu_serves_from_files(tmp_path):
    """Tables and adapters loaded from PLT1 / ADP1 files serve exactly what array uploads serve."""
    from paper_2504_17449_b200 import engine as E

    g = np.load(GOLD)
    cfg = oracle.Config(*[int(x) for x in g["cfg"]])
    mc = E.model_config(*oracle.astuple(cfg))
    R, LABELS, n = 8, 5, len(g["lens"])
    paths = []
    for v in (0, 1):
        t = {k: g[f"t{v}_{k}"] for k in ("key_len", "keys", "freq", "reps")}
        p = str(tmp_path / f"t{v}.plt1")
        plot.save_plt1(t, p, v, int(g[f"t{v}_parent"][0]), "", 0)
        paths.append(p)
    outs = []
    for from_files in (False, True):
        eng = E.GpuEngine(mc, E.generate_higher(mc), max_batch=n, max_seq=g["tokens"].shape[1],
                          bottleneck=R, max_labels=LABELS, max_tasks=n, max_versions=8)
        for v in (0, 1):
            if from_files:
                eng.upload_plt1(paths[v])
            else:
                eng.upload_table(v, int(g[f"t{v}_parent"][0]), g[f"t{v}_key_len"], g[f"t{v}_keys"],
                                 g[f"t{v}_reps"])
        for i in range(n):
            body = E.generate_adapter(mc, R, 1000 + i)
            if from_files:
                p = str(tmp_path / f"a{i}.adp1")
                _write_adp1(p, f"task{i}", body, cfg.hidden_size, R)
                eng.register_task_file(i, p)
            else:
                eng.register_task(i, body)
            w, b = E.generate_head(cfg.hidden_size, LABELS, 2_000_000 + i)
            eng.register_head(i, 0, w, b)
            eng.bind_instance(i, int(g["versions"][i]), i, i)
        outs.append(eng.infer_batch(np.arange(n), g["tokens"], g["lens"]))
        eng.close()
    assert np.array_equal(outs[0].scores, outs[1].scores)


def _write_adp1(path, task_id, body, d, r):
    with open(path, "wb") as f:
        f.write(b"ADP1")
        f.write(len(task_id).to_bytes(4, "little") + task_id.encode())
        f.write(body.shape[0].to_bytes(4, "little") + d.to_bytes(4, "little") + r.to_bytes(4, "little"))
        f.write(np.ascontiguousarray(body, np.float32).tobytes())


def _big_table(seed, n, d, vocab, ngram=3):
    """n distinct keys of length 2..ngram with random f32 reps (a multi-chunk PLT1 at d=128)."""
    rng = np.random.default_rng(seed)
    kl = rng.integers(2, ngram + 1, n).astype(np.uint32)
    keys = np.zeros((n, ngram), np.uint32)
    seen, i = set(), 0
    while i < n:
        k = tuple(int(x) for x in rng.integers(0, vocab, kl[i]))
        if k in seen:
            continue
        seen.add(k)
        keys[i, :kl[i]] = k
        i += 1
    reps = rng.standard_normal((int(kl.sum()), d)).astype(np.float32)
    return {"key_len": kl, "keys": keys, "freq": np.ones(n, np.uint64), "reps": reps}, seen


@pytest.mark.gpu
def test_gpu_streamed_plt1_multi_chunk(tmp_path):
    """hmi_gpu_upload_plt1 over a table larger than its 64 MiB chunk: the gathered rows (h0, f64
    bit pattern) equal those of the array upload; corrupt files fail closed (FormatError, the
    version stays free and a good upload of it then succeeds)."""
    from paper_2504_17449_b200 import engine as E
    from paper_2504_17449_b200._native import DimensionError

    cfg = oracle.Config(128, 2, 2, 2, 256, 5000, 0, 3, 9)
    mc = E.model_config(*oracle.astuple(cfg))
    root = {"key_len": np.ones(5000, np.uint32),
            "keys": np.stack([np.arange(5000), np.zeros(5000), np.zeros(5000)], 1).astype(np.uint32),
            "reps": np.random.default_rng(2).standard_normal((5000, 128)).astype(np.float32)}
    big, seen = _big_table(3, 90_000, 128, 5000)  # ~180k rows x 512 B = ~92 MB of reps
    p = str(tmp_path / "big.plt1")
    plot.save_plt1(big, p, 1, 0, "big", 5000)
    assert os.path.getsize(p) > (64 << 20)
    rng = np.random.default_rng(4)
    n, S = 16, 128
    toks = np.zeros((n, S), np.uint32)
    lens = np.full(n, 60, np.uint32)
    hot = [k for k in list(seen)[:400] if len(k) == 3]
    for i in range(n):
        toks[i, :60] = rng.integers(0, 2000, 60)
        for j in range(0, 57, 6):
            toks[i, j:j + 3] = hot[int(rng.integers(0, len(hot)))]
    h0s = []
    for streamed in (False, True):
        eng = E.GpuEngine(mc, E.generate_higher(mc), max_batch=n, max_seq=S, bottleneck=8,
                          max_labels=5, max_tasks=1, max_versions=4)
        eng.upload_table(0, 0xFFFFFFFF, root["key_len"], root["keys"], root["reps"])
        if streamed:
            # fail-closed: a truncated copy is rejected and leaves version 1 free
            bad = str(tmp_path / "trunc.plt1")
            _corrupt(p, bad, lambda b: b[:-100])
            with pytest.raises(FormatError):
                eng.upload_plt1(bad)
            assert eng.upload_plt1(p) == (1, 0)
        else:
            eng.upload_table(1, 0, big["key_len"], big["keys"], big["reps"])
        eng.register_task(0, E.generate_adapter(mc, 8, 1))
        eng.register_head(0, 0, *E.generate_head(128, 5, 2))
        eng.bind_instance(0, 1, 0, 0)
        eng.set_debug(1)
        eng.infer_batch(np.zeros(n, np.uint32), toks, lens)
        h0s.append(eng.debug_h0(n, S))
        rows, lev = eng.debug_gather(n)
        assert (lev[:, :60] == 1).sum() > 0  # the branch is hit
        eng.close()
    assert np.array_equal(h0s[0].view(np.uint64), h0s[1].view(np.uint64))
    # header checks: wrong hidden size -> DimensionError
    small = str(tmp_path / "d64.plt1")
    t = {k: v for k, v in big.items()}
    t["reps"] = t["reps"][:, :64].copy()
    plot.save_plt1(t, small, 2, 0, "", 0)
    eng = E.GpuEngine(mc, E.generate_higher(mc), max_batch=n, max_seq=S, bottleneck=8,
                      max_labels=5, max_tasks=1, max_versions=4)
    eng.upload_table(0, 0xFFFFFFFF, root["key_len"], root["keys"], root["reps"])
    with pytest.raises(DimensionError):
        eng.upload_plt1(small)
    eng.close()


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["magic", "truncated", "trailing", "zero_freq", "key_len0",
                                  "key_len_big", "duplicate"])
def test_gpu_streamed_plt1_format_errors(tmp_path, case):
    """The streamed reader rejects exactly the files the reference's plot::load rejects."""
    from paper_2504_17449_b200 import engine as E

    g = np.load(GOLD)
    cfg = oracle.Config(*[int(x) for x in g["cfg"]])
    mc = E.model_config(*oracle.astuple(cfg))
    t = _golden_table()
    good = str(tmp_path / "good.plt1")
    plot.save_plt1(t, good, 1, 0, "", 0)
    d = t["reps"].shape[1]
    e0 = 4 + 4 + 4 + 4 + 4 + 4 + 4 + 4
    k0 = int(t["key_len"][0])
    e1 = e0 + 4 + 4 * k0 + 8 + 4 * k0 * d

    def edit(b):
        if case == "magic":
            b[0:4] = b"PLT2"
        elif case == "truncated":
            b = b[:-7]
        elif case == "trailing":
            b += b"\0"
        elif case == "zero_freq":
            b[e0 + 4 + 4 * k0:e0 + 12 + 4 * k0] = (0).to_bytes(8, "little")
        elif case == "key_len0":
            b[e0:e0 + 4] = (0).to_bytes(4, "little")
        elif case == "key_len_big":
            b[e0:e0 + 4] = (9).to_bytes(4, "little")
        elif case == "duplicate":
            b[e1:e1 + 4 + 4 * k0] = b[e0:e0 + 4 + 4 * k0]
        return b

    bad = str(tmp_path / f"{case}.plt1")
    _corrupt(good, bad, edit)
    eng = E.GpuEngine(mc, E.generate_higher(mc), max_batch=4, max_seq=128, bottleneck=8,
                      max_labels=5, max_tasks=1, max_versions=4)
    eng.upload_table(0, 0xFFFFFFFF, g["t0_key_len"], g["t0_keys"], g["t0_reps"])
    with pytest.raises(FormatError):
        eng.upload_plt1(bad)
    assert eng.upload_plt1(good) == (1, 0)  # nothing of the failed attempt was committed
    eng.close()


@pytest.mark.gpu
def test_gpu_bulk_registration(tmp_path):
    """register_tasks / register_task_files (threads) register exactly what register_task does
    (served scores bit-identical), all-or-nothing on conflicts, bad dimensions, bad files."""
    from paper_2504_17449_b200 import engine as E
    from paper_2504_17449_b200._native import ConflictError, DimensionError
    from tests.world import World

    cfg = oracle.Config(128, 2, 2, 2, 256, 300, 0, 3, 5)
    n = 40
    w = World(cfg, n_tasks=n, r=8, labels=5)  # per-task register_task
    inst, toks, lens = w.requests(5, 32, 60)
    want = w.eng.infer_batch(inst, toks, lens)
    mc = E.model_config(*oracle.astuple(cfg))
    paths = []
    for t in range(n):
        p = str(tmp_path / f"t{t}.adp1")
        plot.save_adp1(p, f"task{t}", w.adapters[t], cfg.hidden_size, 8)
        paths.append(p)
    for mode in ("arrays", "files"):
        eng = E.GpuEngine(mc, w.higher, max_batch=32, max_seq=128, bottleneck=8, max_labels=5,
                          max_tasks=n, max_versions=8)
        for t in w.tables:
            eng.upload_table(t["version"], t["parent"], t["key_len"], t["keys"], t["reps"])
        if mode == "arrays":
            with pytest.raises(ConflictError):  # repeated index: nothing registered
                eng.register_tasks([0, 1, 1], [w.adapters[0], w.adapters[1], w.adapters[1]])
            eng.register_tasks(range(n), w.adapters, threads=7)
        else:
            bad = str(tmp_path / "r16.adp1")
            plot.save_adp1(bad, "x", E.generate_adapter(mc, 16, 1), cfg.hidden_size, 16)
            with pytest.raises(DimensionError):
                eng.register_task_files([0, 1], [paths[0], bad])
            trunc = str(tmp_path / "trunc.adp1")
            _corrupt(paths[3], trunc, lambda b: b[:-5])
            with pytest.raises(FormatError):
                eng.register_task_files([2, 3], [paths[2], trunc])
            eng.register_task_files(range(n), paths)  # indices 0..3 are still free
        with pytest.raises(ConflictError):
            eng.register_tasks([5], [w.adapters[5]])
        for t in range(n):
            eng.register_head(t, 0, *w.heads[t])
            eng.bind_instance(t, int(w.inst_version[t]), t, t)
        got = eng.infer_batch(inst, toks, lens)
        assert np.array_equal(got.scores, want.scores), mode
        eng.close()
    w.eng.close()


@pytest.mark.gpu
def test_gpu_streamed_plt1_empty_branch(tmp_path):
    """An empty branch (derive_branch at alpha 0 keeps no keys) streams in as a valid version:
    requests routed to it retrieve through its parent exactly as through the parent itself."""
    from paper_2504_17449_b200 import engine as E

    g = np.load(GOLD)
    cfg = oracle.Config(*[int(x) for x in g["cfg"]])
    mc = E.model_config(*oracle.astuple(cfg))
    empty = {"key_len": np.zeros(0, np.uint32), "keys": np.zeros((0, 3), np.uint32),
             "freq": np.zeros(0, np.uint64), "reps": np.zeros((0, cfg.hidden_size), np.float32)}
    p = str(tmp_path / "empty.plt1")
    plot.save_plt1(empty, p, 1, 0, "odd-label", 0)
    n = len(g["lens"])
    outs = []
    for version in (0, 1):
        eng = E.GpuEngine(mc, E.generate_higher(mc), max_batch=n, max_seq=g["tokens"].shape[1],
                          bottleneck=8, max_labels=5, max_tasks=1, max_versions=4)
        eng.upload_table(0, 0xFFFFFFFF, g["t0_key_len"], g["t0_keys"], g["t0_reps"])
        assert eng.upload_plt1(p) == (1, 0)
        eng.register_task(0, E.generate_adapter(mc, 8, 3))
        eng.register_head(0, 0, *E.generate_head(cfg.hidden_size, 5, 4))
        eng.bind_instance(0, version, 0, 0)
        outs.append(eng.infer_batch(np.zeros(n, np.uint32), g["tokens"], g["lens"]).scores)
        eng.close()
    assert np.array_equal(outs[0], outs[1])
