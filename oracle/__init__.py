# SPDX-License-Identifier: Apache-2.0
"""TEST INFRASTRUCTURE ONLY — the CPU oracle.

Two libraries, both loaded with ctypes:

* ``_build/liboracle.so`` — our plain-C restatement of the reference hot path
  (``hmi_oracle.c``; every function cites the reference file:line it follows).
* ``_ref/libhmiref.so`` — the reference itself, compiled from
  ``/root/reference/proj/src`` by ``build_ref.sh``, driven by ``ref_driver.cpp``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu-baseline /
``--impl reference`` legs may import this package. The product
(``paper_2504_17449_b200``) never does.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, astuple

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libhmiref.so")
REFERENCE_SRC = os.environ.get("HMI_REFERENCE", "/root/reference/proj")

u32p = ctypes.POINTER(ctypes.c_uint32)
i32p = ctypes.POINTER(ctypes.c_int32)
i64p = ctypes.POINTER(ctypes.c_int64)
u64p = ctypes.POINTER(ctypes.c_uint64)
f32p = ctypes.POINTER(ctypes.c_float)
f64p = ctypes.POINTER(ctypes.c_double)


def ptr(a, t):
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"], "array must be C-contiguous"
    return a.ctypes.data_as(t)


@dataclass
class Config:
    """ModelConfig (proj/include/hmi/transformer/config.hpp:10-24)."""

    hidden_size: int = 32
    heads: int = 4
    lower_layers: int = 6
    higher_layers: int = 6
    ffn_size: int = 64
    vocab_size: int = 1024
    mode: int = 0  # 0 encoder, 1 causal
    max_fragment: int = 3
    seed: int = 7

    def c(self):
        return (ctypes.c_uint32 * 9)(*astuple(self))

    def layer_floats(self) -> int:
        d, f = self.hidden_size, self.ffn_size
        return 4 * (d * d + d) + (d * f + f) + (f * d + d) + 4 * d

    def adapter_layer_floats(self, r: int) -> int:
        d = self.hidden_size
        return d * r + r + r * d + d


# Configs of BASELINE.json.
TINY = Config(256, 4, 2, 2, 1024, 1024, 0, 3, 7)          # C1
BASE = Config(768, 12, 6, 6, 3072, 30522, 0, 3, 7)        # C2 / C4
LARGE = Config(1024, 16, 12, 12, 4096, 30522, 0, 3, 7)    # C5
GPT2S = Config(768, 12, 6, 6, 3072, 50257, 1, 3, 7)       # C3


def build_oracle() -> None:
    if not os.path.exists(ORACLE_SO) or os.path.getmtime(ORACLE_SO) < os.path.getmtime(
            os.path.join(HERE, "hmi_oracle.c")):
        subprocess.run(["make", "-s", "-C", HERE], check=True)


def build_ref() -> bool:
    """Builds oracle/_ref from the reference sources when they are present."""
    if os.path.isdir(os.path.join(REFERENCE_SRC, "src")):
        drv = os.path.join(HERE, "ref_driver.cpp")
        if not os.path.exists(REF_SO) or os.path.getmtime(REF_SO) < os.path.getmtime(drv):
            subprocess.run(["bash", os.path.join(HERE, "build_ref.sh")], check=True,
                           stdout=subprocess.DEVNULL)
    return os.path.exists(REF_SO)


_orc = None
_ref = None


def orc() -> ctypes.CDLL:
    global _orc
    if _orc is None:
        build_oracle()
        L = ctypes.CDLL(ORACLE_SO)
        L.orc_layer_floats.restype = ctypes.c_size_t
        L.orc_adapter_layer_floats.restype = ctypes.c_size_t
        L.orc_tree_create.restype = ctypes.c_void_p
        L.orc_tree_create.argtypes = [ctypes.c_uint32, ctypes.c_uint32]
        L.orc_tree_destroy.argtypes = [ctypes.c_void_p]
        L.orc_tree_add_table.argtypes = [ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint32,
                                         ctypes.c_uint32, u32p, u32p, f32p]
        L.orc_retrieve.argtypes = [ctypes.c_void_p, ctypes.c_uint32, u32p, ctypes.c_uint32,
                                   ctypes.c_int, f64p, i64p, u32p, u32p]
        L.orc_higher_forward.argtypes = [ctypes.c_void_p, f32p, f64p, ctypes.c_size_t,
                                         ctypes.c_size_t, f32p, ctypes.c_uint32, f32p, f32p,
                                         ctypes.c_uint32, ctypes.c_int, f64p, i32p, i32p]
        L.orc_lower_forward.argtypes = [ctypes.c_void_p, f32p, f32p, f32p, u32p, ctypes.c_size_t,
                                         f64p]
        L.orc_infer_one.argtypes = [ctypes.c_void_p, f32p, ctypes.c_void_p, ctypes.c_uint32,
                                    u32p, ctypes.c_uint32, ctypes.c_uint32, f32p,
                                    ctypes.c_uint32, f32p, f32p, ctypes.c_uint32, ctypes.c_int,
                                    f64p, i32p, i32p]
        _orc = L
    return _orc


def ref() -> ctypes.CDLL | None:
    global _ref
    if _ref is None:
        if not build_ref():
            return None
        L = ctypes.CDLL(REF_SO)
        vp = ctypes.c_void_p
        L.ref_last_error.restype = ctypes.c_char_p
        L.ref_active_kernels.restype = ctypes.c_char_p
        L.ref_model_generate.restype = vp
        L.ref_model_load.restype = vp
        L.ref_model_free.argtypes = [vp]
        L.ref_model_higher_f32.argtypes = [vp, f32p]
        L.ref_model_embeddings_f32.argtypes = [vp, f32p, f32p]
        L.ref_model_save.argtypes = [vp, ctypes.c_char_p]
        L.ref_adapter_generate.restype = vp
        L.ref_adapter_generate.argtypes = [ctypes.c_char_p, vp, ctypes.c_uint32, ctypes.c_uint64]
        L.ref_adapter_free.argtypes = [vp]
        L.ref_adapter_f32.argtypes = [vp, f32p]
        L.ref_head_generate.restype = vp
        L.ref_head_generate.argtypes = [ctypes.c_char_p, ctypes.c_uint32, ctypes.c_uint32, vp,
                                        ctypes.c_uint64]
        L.ref_head_free.argtypes = [vp]
        L.ref_head_f32.argtypes = [vp, f32p, f32p]
        L.ref_tree_create.restype = vp
        L.ref_tree_create.argtypes = [ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, u32p,
                                      u32p, f32p, u64p]
        L.ref_tree_free.argtypes = [vp]
        L.ref_tree_add_branch.restype = ctypes.c_int64
        L.ref_tree_add_branch.argtypes = [vp, ctypes.c_uint32, ctypes.c_uint32, u32p, u32p, f32p,
                                          u64p]
        L.ref_plt1_load.argtypes = [ctypes.c_char_p, u32p, u32p, u32p, f32p, u64p]
        L.ref_adp1_check.argtypes = [ctypes.c_char_p]
        L.ref_hmi1_check.argtypes = [ctypes.c_char_p]
        L.ref_model_save.argtypes = [vp, ctypes.c_char_p]
        L.ref_adapter_save.argtypes = [vp, ctypes.c_char_p]
        L.ref_plot_persist.argtypes = [vp, ctypes.c_uint32, ctypes.c_char_p]
        L.ref_tree_build_root.restype = vp
        L.ref_tree_build_root.argtypes = [vp, ctypes.c_uint32, u32p, u32p]
        L.ref_tree_derive_branch.restype = ctypes.c_int64
        L.ref_tree_derive_branch.argtypes = [vp, vp, ctypes.c_uint32, u32p, u32p,
                                             ctypes.c_double]
        L.ref_tree_table_size.restype = ctypes.c_int64
        L.ref_tree_table_size.argtypes = [vp, ctypes.c_uint32, u64p]
        L.ref_tree_table_export.argtypes = [vp, ctypes.c_uint32, u32p, u32p, f32p, u64p, u32p]
        L.ref_retrieve.argtypes = [vp, ctypes.c_uint32, u32p, ctypes.c_uint32, ctypes.c_uint32,
                                   f64p, u32p]
        L.ref_infer.argtypes = [vp, vp, ctypes.c_uint32, u32p, ctypes.POINTER(vp),
                                ctypes.POINTER(vp), u32p, u32p, ctypes.c_uint32,
                                ctypes.c_uint32, f64p, i32p, i32p, ctypes.c_uint32]
        L.ref_pool_create.restype = vp
        L.ref_pool_create.argtypes = [ctypes.c_uint64]
        L.ref_pool_free.argtypes = [vp]
        L.ref_pool_register.argtypes = [vp, ctypes.c_char_p, ctypes.c_uint32, ctypes.c_uint32,
                                        ctypes.c_uint32]
        L.ref_pool_op.restype = ctypes.c_int64
        L.ref_pool_op.argtypes = [vp, ctypes.c_int, ctypes.c_uint32,
                                  ctypes.POINTER(ctypes.c_char_p), ctypes.c_uint32, i32p, u64p,
                                  ctypes.c_char_p, ctypes.c_uint64]
        L.ref_pool_stats.argtypes = [vp, u64p]
        _ref = L
    return _ref


# ---------------------------------------------------------------------------
# restatement (liboracle)
# ---------------------------------------------------------------------------
def generate_model(cfg: Config, lower: bool = False):
    """generate_model (weights.cpp:72-88): returns dict of f32 arrays."""
    L = orc()
    d = cfg.hidden_size
    lf = cfg.layer_floats()
    tok = np.empty((cfg.vocab_size, d), np.float32)
    pos = np.empty((cfg.max_fragment, d), np.float32)
    low = np.empty((cfg.lower_layers, lf), np.float32) if lower else None
    hi = np.empty((cfg.higher_layers, lf), np.float32)
    rc = L.orc_generate_model(ctypes.byref(cfg.c()), ptr(tok, f32p), ptr(pos, f32p),
                              ptr(low, f32p), ptr(hi, f32p))
    assert rc == 0
    return {"token_embedding": tok, "position_embedding": pos, "lower": low, "higher": hi}


def generate_higher(cfg: Config) -> np.ndarray:
    L = orc()
    hi = np.empty((cfg.higher_layers, cfg.layer_floats()), np.float32)
    rc = L.orc_generate_model(ctypes.byref(cfg.c()), None, None, None, ptr(hi, f32p))
    assert rc == 0
    return hi


def generate_adapter(cfg: Config, r: int, seed: int) -> np.ndarray:
    """generate_adapter_set (adapter_set.cpp:15-25): [layers, adapter_layer_floats]."""
    out = np.empty((cfg.higher_layers, cfg.adapter_layer_floats(r)), np.float32)
    rc = orc().orc_generate_adapter(ctypes.byref(cfg.c()), ctypes.c_uint32(r),
                                    ctypes.c_uint64(seed), ptr(out, f32p))
    assert rc == 0
    return out


def generate_head(d: int, labels: int, seed: int):
    """generate_output_head (weights.cpp:105-118): (w [d x labels], b [labels])."""
    w = np.empty((d, labels), np.float32)
    b = np.empty((labels,), np.float32)
    rc = orc().orc_generate_head(ctypes.c_uint32(d), ctypes.c_uint32(labels),
                                 ctypes.c_uint64(seed), ptr(w, f32p), ptr(b, f32p))
    assert rc == 0
    return w, b


class OracleTree:
    """VersionTree restatement: tables added in order; global rep rows numbered
    in upload order (table, entry, row)."""

    def __init__(self, ngram: int, d: int):
        self.ngram, self.d = ngram, d
        self.h = orc().orc_tree_create(ngram, d)

    def __del__(self):
        if getattr(self, "h", None):
            orc().orc_tree_destroy(self.h)
            self.h = None

    def add_table(self, version: int, parent: int, key_len, keys, reps) -> None:
        key_len = np.ascontiguousarray(key_len, np.uint32)
        keys = np.ascontiguousarray(keys, np.uint32).reshape(-1, self.ngram)
        reps = np.ascontiguousarray(reps, np.float32)
        rc = orc().orc_tree_add_table(self.h, version, parent & 0xFFFFFFFF, len(key_len),
                                      ptr(key_len, u32p), ptr(keys, u32p), ptr(reps, f32p))
        if rc:
            raise RuntimeError(f"orc_tree_add_table failed: {rc}")

    def retrieve(self, version: int, tokens, mode: int):
        tokens = np.ascontiguousarray(tokens, np.uint32)
        n = len(tokens)
        out = np.empty((n, self.d), np.float64)
        gather = np.empty((n, self.ngram), np.int64)
        levels = np.empty((n, self.ngram), np.uint32)
        srcs = np.empty((n, self.ngram), np.uint32)
        rc = orc().orc_retrieve(self.h, version, ptr(tokens, u32p), n, mode, ptr(out, f64p),
                                ptr(gather, i64p), ptr(levels, u32p), ptr(srcs, u32p))
        if rc:
            raise RuntimeError(f"orc_retrieve failed: {rc}")
        return out, gather, levels, srcs


def higher_forward(cfg: Config, higher: np.ndarray, h: np.ndarray, valid_len: int,
                   adapters: np.ndarray | None, r: int, head_w, head_b, head_kind: int = 0):
    """higher_stack_forward + apply_head on one request (model.cpp:84-185)."""
    h = np.ascontiguousarray(h, np.float64).copy()
    labels = head_b.shape[0]
    scores = np.zeros(labels, np.float64)
    label = ctypes.c_int32(-1)
    tags = np.zeros(h.shape[0], np.int32)
    ad = None if adapters is None else np.ascontiguousarray(adapters, np.float32)
    rc = orc().orc_higher_forward(ctypes.byref(cfg.c()), ptr(np.ascontiguousarray(higher), f32p),
                                  ptr(h, f64p), h.shape[0], valid_len, ptr(ad, f32p), r,
                                  ptr(np.ascontiguousarray(head_w), f32p),
                                  ptr(np.ascontiguousarray(head_b), f32p), labels, head_kind,
                                  ptr(scores, f64p), ctypes.byref(label), ptr(tags, i32p))
    assert rc == 0
    return scores, label.value, tags[:valid_len], h


def lower_forward(cfg: Config, model: dict, tokens) -> np.ndarray:
    """lower_stack_forward (model.cpp:96-118) of one fragment: [len x d] f64 PLOT rep rows.
    `model` is generate_model(cfg, lower=True)."""
    tokens = np.ascontiguousarray(tokens, np.uint32)
    out = np.empty((len(tokens), cfg.hidden_size), np.float64)
    rc = orc().orc_lower_forward(ctypes.byref(cfg.c()), ptr(model["token_embedding"], f32p),
                                 ptr(model["position_embedding"], f32p), ptr(model["lower"], f32p),
                                 ptr(tokens, u32p), len(tokens), ptr(out, f64p))
    assert rc == 0, rc
    return out


def _kgram_counts(corpus, k: int) -> dict:
    """count_kgrams (table.cpp:16-27): occurrences of every k-gram over the corpus."""
    counts: dict = {}
    for seq in corpus:
        seq = [int(x) for x in seq]
        for i in range(len(seq) - k + 1):
            key = tuple(seq[i:i + k])
            counts[key] = counts.get(key, 0) + 1
    return counts


def plot_select_root(corpus, ngram: int, vocab: int) -> list:
    """build_root's entries (table.cpp:29-58) as (key, freq) in std::map key order: every
    k-gram (k = 1..ngram) with its count, then every vocabulary uni-gram absent from the
    corpus with frequency 1. Python tuple order = std::vector<uint32_t> lexicographic order."""
    if len(corpus) == 0:
        raise ValueError("cannot build a table from an empty corpus")
    entries: dict = {}
    for k in range(1, ngram + 1):
        for key, n in _kgram_counts(corpus, k).items():
            entries.setdefault(key, n)
    for t in range(vocab):
        entries.setdefault((t,), 1)
    return sorted(entries.items())


def plot_select_branch(corpus, ngram: int, alpha_percent: float) -> list:
    """derive_branch's entries (table.cpp:60-104): the corpus' ngram-grams by count
    descending (ties in key order, stable sort) until cumulative * 10000 >= round(alpha *
    100) * total; returned in key order."""
    if not 0.0 <= alpha_percent <= 100.0:
        raise ValueError("alpha_percent must be in [0, 100]")
    alpha_centi = int(np.floor(alpha_percent * 100.0 + 0.5))  # std::llround, alpha >= 0
    counts = _kgram_counts(corpus, ngram)
    total = sum(counts.values())
    if total == 0 or alpha_centi == 0:
        return []
    order = sorted(sorted(counts.items()), key=lambda kv: -kv[1])
    out, cum = [], 0
    for key, n in order:
        cum += n
        out.append((key, n))
        if cum * 10000 >= alpha_centi * total:
            break
    return sorted(out)


def infer_one(cfg: Config, higher, tree: OracleTree, version: int, tokens, adapters, r: int,
              head_w, head_b, head_kind: int = 0):
    tokens = np.ascontiguousarray(tokens, np.uint32)
    labels = head_b.shape[0]
    scores = np.zeros(labels, np.float64)
    label = ctypes.c_int32(-1)
    tags = np.zeros(len(tokens), np.int32)
    ad = None if adapters is None else np.ascontiguousarray(adapters, np.float32)
    rc = orc().orc_infer_one(ctypes.byref(cfg.c()), ptr(np.ascontiguousarray(higher), f32p),
                             tree.h, version, ptr(tokens, u32p), len(tokens), len(tokens),
                             ptr(ad, f32p), r, ptr(np.ascontiguousarray(head_w), f32p),
                             ptr(np.ascontiguousarray(head_b), f32p), labels, head_kind,
                             ptr(scores, f64p), ctypes.byref(label), ptr(tags, i32p))
    assert rc == 0, rc
    return scores, label.value, tags


# ---------------------------------------------------------------------------
# the reference itself (libhmiref)
# ---------------------------------------------------------------------------
class RefModel:
    def __init__(self, cfg: Config):
        self.cfg = cfg
        self.h = ref().ref_model_generate(ctypes.byref(cfg.c()))
        assert self.h, ref().ref_last_error()

    def __del__(self):
        if getattr(self, "h", None) and _ref is not None:
            _ref.ref_model_free(self.h)
            self.h = None

    def higher(self) -> np.ndarray:
        out = np.empty((self.cfg.higher_layers, self.cfg.layer_floats()), np.float32)
        assert ref().ref_model_higher_f32(self.h, ptr(out, f32p)) == 0
        return out


class RefTree:
    def __init__(self, ngram, d, key_len, keys, reps, freq=None, handle=None):
        self.ngram, self.d = ngram, d
        if handle is not None:
            self.h = handle
            return
        key_len = np.ascontiguousarray(key_len, np.uint32)
        keys = np.ascontiguousarray(keys, np.uint32)
        reps = np.ascontiguousarray(reps, np.float32)
        fq = None if freq is None else np.ascontiguousarray(freq, np.uint64)
        self.h = ref().ref_tree_create(ngram, d, len(key_len), ptr(key_len, u32p),
                                       ptr(keys, u32p), ptr(reps, f32p), ptr(fq, u64p))
        assert self.h, ref().ref_last_error()

    def __del__(self):
        if getattr(self, "h", None) and _ref is not None:
            _ref.ref_tree_free(self.h)
            self.h = None

    def add_branch(self, parent, key_len, keys, reps, freq=None) -> int:
        key_len = np.ascontiguousarray(key_len, np.uint32)
        keys = np.ascontiguousarray(keys, np.uint32)
        reps = np.ascontiguousarray(reps, np.float32)
        fq = None if freq is None else np.ascontiguousarray(freq, np.uint64)
        v = ref().ref_tree_add_branch(self.h, parent, len(key_len), ptr(key_len, u32p),
                                      ptr(keys, u32p), ptr(reps, f32p), ptr(fq, u64p))
        assert v >= 0, ref().ref_last_error()
        return int(v)

    def export(self, version: int):
        rows = ctypes.c_uint64(0)
        n = ref().ref_tree_table_size(self.h, version, ctypes.byref(rows))
        assert n >= 0
        key_len = np.empty(n, np.uint32)
        keys = np.empty((n, self.ngram), np.uint32)
        reps = np.empty((rows.value, self.d), np.float32)
        freq = np.empty(n, np.uint64)
        parent = ctypes.c_uint32(0)
        assert ref().ref_tree_table_export(self.h, version, ptr(key_len, u32p), ptr(keys, u32p),
                                           ptr(reps, f32p), ptr(freq, u64p),
                                           ctypes.byref(parent)) == 0
        return key_len, keys, reps, freq, parent.value

    def retrieve(self, version, tokens, mode):
        tokens = np.ascontiguousarray(tokens, np.uint32)
        out = np.empty((len(tokens), self.d), np.float64)
        levels = np.empty((len(tokens), self.ngram), np.uint32)
        rc = ref().ref_retrieve(self.h, version, ptr(tokens, u32p), len(tokens), mode,
                                ptr(out, f64p), ptr(levels, u32p))
        assert rc == 0, ref().ref_last_error()
        return out, levels


def ref_set_kernels(name: str) -> None:
    assert ref().ref_set_kernels(name.encode()) == 0


class RefTask:
    """AdapterSet + OutputHead generated by the reference's own generators."""

    def __init__(self, cfg: Config, task_id: str, r: int, seed: int, labels: int,
                 head_seed: int, head_kind: int = 0):
        L = ref()
        self.adapter = L.ref_adapter_generate(task_id.encode(), ctypes.byref(cfg.c()), r, seed)
        self.head = L.ref_head_generate(task_id.encode(), head_kind, labels,
                                        ctypes.byref(cfg.c()), head_seed)
        assert self.adapter and self.head, L.ref_last_error()
        self.cfg, self.r, self.labels = cfg, r, labels

    def __del__(self):
        if _ref is not None:
            if getattr(self, "adapter", None):
                _ref.ref_adapter_free(self.adapter)
            if getattr(self, "head", None):
                _ref.ref_head_free(self.head)

    def adapter_f32(self):
        out = np.empty((self.cfg.higher_layers, self.cfg.adapter_layer_floats(self.r)), np.float32)
        assert ref().ref_adapter_f32(self.adapter, ptr(out, f32p)) == 0
        return out

    def head_f32(self):
        w = np.empty((self.cfg.hidden_size, self.labels), np.float32)
        b = np.empty((self.labels,), np.float32)
        assert ref().ref_head_f32(self.head, ptr(w, f32p), ptr(b, f32p)) == 0
        return w, b


def ref_infer(model: RefModel, tree: RefTree, versions, tasks, tokens, lens, max_labels: int,
              threads: int = 1):
    """retrieve_sequence + higher_stack_forward per request, `threads` host threads."""
    n = len(versions)
    versions = np.ascontiguousarray(versions, np.uint32)
    tokens = np.ascontiguousarray(tokens, np.uint32)
    lens = np.ascontiguousarray(lens, np.uint32)
    sets = (ctypes.c_void_p * n)(*[t.adapter for t in tasks])
    heads = (ctypes.c_void_p * n)(*[t.head for t in tasks])
    scores = np.zeros((n, max_labels), np.float64)
    labels = np.zeros(n, np.int32)
    rc = ref().ref_infer(model.h, tree.h, n, ptr(versions, u32p), sets, heads,
                         ptr(tokens, u32p), ptr(lens, u32p), tokens.shape[1], max_labels,
                         ptr(scores, f64p), ptr(labels, i32p), None, threads)
    assert rc == 0, ref().ref_last_error()
    return scores, labels
