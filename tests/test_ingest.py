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
