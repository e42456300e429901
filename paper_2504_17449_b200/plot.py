# SPDX-License-Identifier: Apache-2.0
"""GPU PLOT builder (host mirror of include/hmi_gpu.h's hmi_plot_* entry points).

Mirrors the reference's offline table construction (proj/src/plot/table.cpp:29-104):
``build_root(corpus, model)`` and ``derive_branch(root, domain_corpus, domain_model, alpha)``,
with lower_stack_forward (proj/src/transformer/model.cpp:96-118) on the B200. Tables come
back as dicts ``{key_len, keys, freq, reps}`` in the reference's std::map entry order, ready
for ``GpuEngine.upload_table``.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _native
from ._native import ModelConfig, check
from .engine import _p, layer_floats

P = ctypes.POINTER


def generate_model(cfg: ModelConfig):
    """generate_model(cfg) (weights.cpp:72-88): token / position embeddings and the lower
    layers (f32, HMI1 per-layer order), seeded exactly as the reference draws them."""
    d = cfg.hidden_size
    tok = np.empty((cfg.vocab_size, d), np.float32)
    pos = np.empty((cfg.max_fragment, d), np.float32)
    low = np.empty((cfg.lower_layers, layer_floats(cfg)), np.float32)
    check(_native.lib().hmi_generate_model(ctypes.byref(cfg), _p(tok, ctypes.c_float),
                                           _p(pos, ctypes.c_float), _p(low, ctypes.c_float), None))
    return tok, pos, low


def _corpus(corpus):
    seqs = [np.ascontiguousarray(s, np.uint32).ravel() for s in corpus]
    lens = np.array([len(s) for s in seqs], np.uint32)
    toks = np.ascontiguousarray(np.concatenate(seqs) if seqs else np.zeros(0, np.uint32), np.uint32)
    return len(seqs), lens, toks


def _finish(h, ngram: int, d: int) -> dict:
    """Read a hmi_plot_table into arrays and free it."""
    L = _native.lib()
    try:
        n = ctypes.c_uint32(0)
        rows = ctypes.c_uint64(0)
        has = ctypes.c_uint32(0)
        check(L.hmi_plot_table_info(h, ctypes.byref(n), ctypes.byref(rows), ctypes.byref(has)))
        key_len = np.empty(n.value, np.uint32)
        keys = np.zeros((n.value, ngram), np.uint32)
        freq = np.empty(n.value, np.uint64)
        reps = np.empty((rows.value, d), np.float32) if has.value else None
        check(L.hmi_plot_table_read(h, _p(key_len, ctypes.c_uint32), _p(keys, ctypes.c_uint32),
                                    _p(freq, ctypes.c_uint64),
                                    _p(reps, ctypes.c_float) if reps is not None else None))
    finally:
        L.hmi_plot_table_free(h)
    return {"key_len": key_len, "keys": keys, "freq": freq, "reps": reps}


def table_handle(t: dict, ngram: int, d: int):
    """A hmi_plot_table from arrays (e.g. a PLT1 file's body); caller frees it."""
    kl = np.ascontiguousarray(t["key_len"], np.uint32)
    ks = np.ascontiguousarray(t["keys"], np.uint32).reshape(len(kl), ngram)
    fq = np.ascontiguousarray(t["freq"], np.uint64)
    reps = t.get("reps")
    rp = None if reps is None else np.ascontiguousarray(reps, np.float32)
    h = ctypes.c_void_p()
    check(_native.lib().hmi_plot_table_create(ngram, d, len(kl), _p(kl, ctypes.c_uint32),
                                              _p(ks, ctypes.c_uint32), _p(fq, ctypes.c_uint64),
                                              _p(rp, ctypes.c_float) if rp is not None else None,
                                              ctypes.byref(h)))
    return h


def load_plt1(path: str):
    """A PLT1 file (plot_io.cpp:35-72) -> (table dict, version_id, parent_id, alpha_centi)."""
    h = ctypes.c_void_p()
    v, p, a = ctypes.c_uint32(0), ctypes.c_uint32(0), ctypes.c_uint32(0)
    check(_native.lib().hmi_plot_table_load(path.encode(), ctypes.byref(h), ctypes.byref(v),
                                            ctypes.byref(p), ctypes.byref(a)))
    return _finish_any(h), v.value, p.value, a.value


def _finish_any(h) -> dict:
    """Like _finish for a handle whose ngram / d only the library knows."""
    ngram, d = ctypes.c_uint32(0), ctypes.c_uint32(0)
    try:
        check(_native.lib().hmi_plot_table_shape(h, ctypes.byref(ngram), ctypes.byref(d)))
    except Exception:
        _native.lib().hmi_plot_table_free(h)
        raise
    return _finish(h, ngram.value, d.value)


def save_plt1(table: dict, path: str, version_id: int, parent_id: int, label: str = "",
              alpha_centi: int = 0, ngram: int | None = None, d: int | None = None) -> None:
    """Persist a table as PLT1 (plot_io.cpp:17-33), readable by the reference's plot::load."""
    ngram = ngram or np.asarray(table["keys"]).shape[1]
    d = d or np.asarray(table["reps"]).shape[1]
    h = table_handle(table, ngram, d)
    try:
        check(_native.lib().hmi_plot_table_save(h, path.encode(), version_id, parent_id & 0xFFFFFFFF,
                                                label.encode(), alpha_centi))
    finally:
        _native.lib().hmi_plot_table_free(h)


def load_adp1(path: str):
    """An ADP1 adapter set (adapter_set.cpp:48-75) -> (task_id, f32 body [layers, floats])."""
    L = _native.lib()
    layers, d, r = ctypes.c_uint32(0), ctypes.c_uint32(0), ctypes.c_uint32(0)
    name = ctypes.create_string_buffer(1024)
    check(L.hmi_adapter_set_load(path.encode(), name, 1024, ctypes.byref(layers), ctypes.byref(d),
                                 ctypes.byref(r), None))
    per = 2 * d.value * r.value + r.value + d.value
    body = np.empty((layers.value, per), np.float32)
    check(L.hmi_adapter_set_load(path.encode(), None, 0, None, None, None, _p(body, ctypes.c_float)))
    return name.value.decode(), body


def save_adp1(path: str, task_id: str, body, d: int, r: int) -> None:
    """ADP1 writer (adapter_set.cpp:27-46): magic, task id, layers, d, r, f32 body."""
    body = np.ascontiguousarray(body, np.float32).reshape(-1, 2 * d * r + r + d)
    name = task_id.encode()
    with open(path, "wb") as f:
        f.write(b"ADP1" + len(name).to_bytes(4, "little") + name)
        for v in (body.shape[0], d, r):
            f.write(int(v).to_bytes(4, "little"))
        f.write(body.tobytes())


def load_hmi1(path: str):
    """An HMI1 model (model_io.cpp:83-115) -> (ModelConfig, token_emb, pos_emb, lower, higher)."""
    L = _native.lib()
    cfg = ModelConfig()
    check(L.hmi_model_load(path.encode(), ctypes.byref(cfg), None, None, None, None))
    d = cfg.hidden_size
    tok = np.empty((cfg.vocab_size, d), np.float32)
    pos = np.empty((cfg.max_fragment, d), np.float32)
    low = np.empty((cfg.lower_layers, layer_floats(cfg)), np.float32)
    hi = np.empty((cfg.higher_layers, layer_floats(cfg)), np.float32)
    check(L.hmi_model_load(path.encode(), ctypes.byref(cfg), _p(tok, ctypes.c_float),
                           _p(pos, ctypes.c_float), _p(low, ctypes.c_float), _p(hi, ctypes.c_float)))
    return cfg, tok, pos, low, hi


def select_root(corpus, ngram: int, vocab: int) -> dict:
    """build_root's key selection only (host, no GPU): keys + frequencies."""
    n_seq, lens, toks = _corpus(corpus)
    h = ctypes.c_void_p()
    check(_native.lib().hmi_plot_select_root(ngram, vocab, n_seq, _p(lens, ctypes.c_uint32),
                                             _p(toks, ctypes.c_uint32), ctypes.byref(h)))
    return _finish(h, ngram, 0)


def select_branch(corpus, ngram: int, alpha_percent: float) -> dict:
    """derive_branch's key selection only (host, no GPU)."""
    n_seq, lens, toks = _corpus(corpus)
    h = ctypes.c_void_p()
    check(_native.lib().hmi_plot_select_branch(ngram, n_seq, _p(lens, ctypes.c_uint32),
                                               _p(toks, ctypes.c_uint32), alpha_percent,
                                               ctypes.byref(h)))
    return _finish(h, ngram, 0)


class GpuPlotBuilder:
    """One model's lower stack on one GPU (hmi_plot_builder)."""

    def __init__(self, cfg: ModelConfig, token_emb=None, pos_emb=None, lower=None, *,
                 device: int = 0, precision: int = 0, max_rows: int = 0):
        if token_emb is None:
            token_emb, pos_emb, lower = generate_model(cfg)
        self.cfg = cfg
        self._keep = [np.ascontiguousarray(x, np.float32) for x in (token_emb, pos_emb, lower)]
        h = ctypes.c_void_p()
        check(_native.lib().hmi_plot_builder_create(
            device, ctypes.byref(cfg), _p(self._keep[0], ctypes.c_float),
            _p(self._keep[1], ctypes.c_float), _p(self._keep[2], ctypes.c_float), precision,
            max_rows, ctypes.byref(h)))
        self.h = h

    def close(self) -> None:
        if self.h:
            _native.lib().hmi_plot_builder_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def forward(self, key_len, keys) -> np.ndarray:
        """lower_stack_forward of each fragment; rows in fragment order [sum(key_len) x d]."""
        kl = np.ascontiguousarray(key_len, np.uint32)
        ks = np.ascontiguousarray(keys, np.uint32).reshape(len(kl), self.cfg.max_fragment)
        out = np.empty((int(kl.sum()), self.cfg.hidden_size), np.float32)
        check(_native.lib().hmi_plot_forward(self.h, len(kl), _p(kl, ctypes.c_uint32),
                                             _p(ks, ctypes.c_uint32), _p(out, ctypes.c_float)))
        return out

    def stats(self) -> tuple[float, int]:
        """(device ms, rows) accumulated over every GPU pass of this builder."""
        ms = ctypes.c_double(0)
        rows = ctypes.c_uint64(0)
        check(_native.lib().hmi_plot_builder_stats(self.h, ctypes.byref(ms), ctypes.byref(rows)))
        return ms.value, rows.value

    def build_root(self, corpus) -> dict:
        n_seq, lens, toks = _corpus(corpus)
        h = ctypes.c_void_p()
        check(_native.lib().hmi_plot_build_root(self.h, n_seq, _p(lens, ctypes.c_uint32),
                                                _p(toks, ctypes.c_uint32), ctypes.byref(h)))
        return _finish(h, self.cfg.max_fragment, self.cfg.hidden_size)

    def derive_branch(self, root: dict, domain_corpus, alpha_percent: float) -> dict:
        """derive_branch with THIS builder's model as the domain model."""
        rt = table_handle(root, self.cfg.max_fragment, self.cfg.hidden_size)
        try:
            n_seq, lens, toks = _corpus(domain_corpus)
            h = ctypes.c_void_p()
            check(_native.lib().hmi_plot_derive_branch(self.h, rt, n_seq, _p(lens, ctypes.c_uint32),
                                                       _p(toks, ctypes.c_uint32), alpha_percent,
                                                       ctypes.byref(h)))
        finally:
            _native.lib().hmi_plot_table_free(rt)
        return _finish(h, self.cfg.max_fragment, self.cfg.hidden_size)
