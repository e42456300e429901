# SPDX-License-Identifier: Apache-2.0
"""Seeded synthetic workloads of BASELINE.json's configs.

PLOT tables are synthetic seeded f32 rows (SPEC.md:676 allows synthetic
tables) keyed exactly as the reference's offline builder would key them:

* root (version 0): the vocabulary-wide uni-gram backstop plus every distinct
  k-gram (k = 1..n) of a general corpus — build_root's enumeration
  (proj/src/plot/table.cpp:29-58);
* one branch per domain: the n-grams of the domain corpus sorted by count
  descending, ties by key, cut at the shortest prefix reaching alpha% of
  occurrences in exact integer arithmetic — derive_branch's selection
  (table.cpp:60-104); optional sub-domain level (C5's 3-level tree).

Requests: tenants uniform at random; 95% of tokens are a
window of the tenant's domain corpus, 5% uniform vocabulary (fallback path).
Seeds: model 7, adapter 1000 + tenant, head 2e6 + tenant, workload 42.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

ADAPTER_SEED = 1000
HEAD_SEED = 2_000_000


@dataclass
class Workload:
    name: str
    hidden_size: int
    heads: int
    lower_layers: int
    higher_layers: int
    ffn_size: int
    vocab_size: int
    mode: int = 0
    max_fragment: int = 3
    model_seed: int = 7
    n_tenants: int = 1000
    n_domains: int = 8
    subdomains: int = 0          # per domain (3-level tree when > 0)
    r: int = 64
    labels: int = 8
    head_kind: int = 0
    batch: int = 256
    seq: int = 128
    seed: int = 42
    domain_vocab: int = 2000
    domain_tokens: int = 65536
    root_tokens: int = 16384
    zipf_s: float = 1.1
    alpha: float = 50.0
    p_noise: float = 0.05
    pool_fraction: float = 1.0   # HBM slot pool as a fraction of all tenants' adapters
    gen_tokens: int = 0          # causal generation: tokens generated per request (C3)

    def flops_per_request(self) -> int:
        """Algorithmic FLOPs: F_layer = 2L(4d^2 + 2df + 2dr) + 4L^2 d,
        F_req = layers * F_layer + 2 d labels (cls head on one row)."""
        L, d, f, r = self.seq, self.hidden_size, self.ffn_size, self.r
        attn = 4 * L * L * d if self.mode == 0 else 2 * L * (L + 1) * d
        layer = 2 * L * (4 * d * d + 2 * d * f + 2 * d * r) + attn
        return self.higher_layers * layer + 2 * d * self.labels

    def generate_flops_per_request(self) -> int:
        """Prompt forward + lm head, then one single-row step per further token at
        context c: layers * (2 (4d^2 + 2df + 2dr) + 4 c d) + 2 d V."""
        L, d, f, r = self.seq, self.hidden_size, self.ffn_size, self.r
        total = self.flops_per_request()
        for k in range(1, self.gen_tokens):
            c = L + k  # keys of the row at position L + k - 1
            total += self.higher_layers * (2 * (4 * d * d + 2 * d * f + 2 * d * r) + 4 * c * d)
            total += 2 * d * self.labels
        return total


CONFIGS = {
    # C1 tiny hBERT (4 layers = 2 PLOT + 2 higher), 16 tenants, batch 32
    "c1": Workload("tiny-hBERT", 256, 4, 2, 2, 1024, 1024, n_tenants=16, n_domains=2, r=16,
                   batch=32, domain_vocab=300, domain_tokens=8192, root_tokens=4096),
    # C2 hBERT-base (12 layers = 6 PLOT + 6 higher), 1,000 tenants, 8 domains, batch 256
    "c2": Workload("hBERT-base", 768, 12, 6, 6, 3072, 30522),
    # C3 hGPT-2 small (causal): prompt 128 + 32 greedy tokens, one shared vocabulary lm head
    "c3": Workload("hGPT-2-small", 768, 12, 6, 6, 3072, 50257, mode=1, head_kind=2,
                   labels=50257, gen_tokens=32),
    # C4 hBERT-base, 10,000 tenants swapped through a bounded HBM slot pool
    "c4": Workload("hBERT-base-10k-swap", 768, 12, 6, 6, 3072, 30522, n_tenants=10000,
                   pool_fraction=0.6),
    # C5 hBERT-large, 10,000 tenants on a 3-level tree
    "c5": Workload("hBERT-large", 1024, 16, 12, 12, 4096, 30522, n_tenants=10000,
                   subdomains=2),
}


def _zipf_probs(m: int, s: float) -> np.ndarray:
    p = 1.0 / np.arange(1, m + 1, dtype=np.float64) ** s
    return p / p.sum()


def _sequences(rng, vocab_ids: np.ndarray, tokens: int, seq: int, s: float) -> np.ndarray:
    n_seq = max(1, tokens // seq)
    p = _zipf_probs(len(vocab_ids), s)
    idx = rng.choice(len(vocab_ids), size=(n_seq, seq), p=p)
    return vocab_ids[idx].astype(np.uint32)


def _encode(grams: np.ndarray, V: int) -> np.ndarray:
    key = np.zeros(grams.shape[0], np.int64)
    for j in range(grams.shape[1]):
        key = key * V + grams[:, j].astype(np.int64)
    return key


def _kgrams(corpus: np.ndarray, k: int) -> np.ndarray:
    """All k-grams of every sequence (count_kgrams, table.cpp:16-27), [N, k]."""
    n_seq, L = corpus.shape
    if L < k:
        return np.zeros((0, k), np.uint32)
    idx = np.arange(L - k + 1)[:, None] + np.arange(k)[None, :]
    return corpus[:, idx].reshape(-1, k)


def _table(rng, version, parent, keys_by_len, ngram, d):
    """keys_by_len: list of [N_k, k] arrays; entries sorted like std::map<vector<u32>>."""
    ks = []
    for arr in keys_by_len:
        for row in arr:
            ks.append(tuple(int(x) for x in row))
    ks.sort()
    key_len = np.array([len(k) for k in ks], np.uint32)
    keys = np.zeros((len(ks), ngram), np.uint32)
    for i, k in enumerate(ks):
        keys[i, :len(k)] = k
    rows = int(key_len.sum())
    reps = rng.standard_normal((rows, d), dtype=np.float32)
    return {"version": version, "parent": parent, "key_len": key_len, "keys": keys, "reps": reps}


def derive_selection(corpus: np.ndarray, n: int, V: int, alpha_percent: float) -> np.ndarray:
    """derive_branch's key selection (table.cpp:60-104), exact integer test."""
    grams = _kgrams(corpus, n)
    if grams.shape[0] == 0:
        return np.zeros((0, n), np.uint32)
    enc = _encode(grams, V)
    uniq, counts = np.unique(enc, return_counts=True)  # ascending key = lexicographic order
    order = np.argsort(-counts, kind="stable")          # count desc, ties by key
    alpha_centi = int(round(alpha_percent * 100))
    total = int(counts.sum())
    if total == 0 or alpha_centi == 0:
        return np.zeros((0, n), np.uint32)
    cum = np.cumsum(counts[order].astype(np.int64))
    cut = int(np.argmax(cum * 10000 >= alpha_centi * total)) + 1
    sel = uniq[order[:cut]]
    out = np.zeros((len(sel), n), np.uint32)
    for j in range(n - 1, -1, -1):
        out[:, j] = sel % V
        sel = sel // V
    return out


class World:
    """Tables, domain corpora and tenant->domain mapping of one workload."""

    def __init__(self, w: Workload):
        self.w = w
        rng = np.random.default_rng(w.seed)
        V, n, d = w.vocab_size, w.max_fragment, w.hidden_size
        # root: general corpus over the whole vocabulary
        root_corpus = _sequences(rng, np.arange(V, dtype=np.uint32), w.root_tokens, w.seq, w.zipf_s)
        root_keys = [np.arange(V, dtype=np.uint32)[:, None]]
        for k in range(2, n + 1):
            g = _kgrams(root_corpus, k)
            root_keys.append(np.unique(g, axis=0) if len(g) else g)
        self.tables = [_table(np.random.default_rng(w.seed * 1000), 0, 0xFFFFFFFF, root_keys, n, d)]
        # domains (and optional sub-domains)
        self.domain_corpus = []
        self.leaf_versions = []
        version = 1
        for dom in range(w.n_domains):
            vocab_ids = rng.choice(V, w.domain_vocab, replace=False).astype(np.uint32)
            corpus = _sequences(rng, vocab_ids, w.domain_tokens, w.seq, w.zipf_s)
            sel = derive_selection(corpus, n, V, w.alpha)
            self.tables.append(_table(np.random.default_rng(w.seed * 1000 + version), version, 0,
                                      [sel], n, d))
            dom_version = version
            version += 1
            if w.subdomains:
                for sub in range(w.subdomains):
                    sub_ids = rng.choice(vocab_ids, w.domain_vocab // 2, replace=False)
                    sc = _sequences(rng, sub_ids, w.domain_tokens // 2, w.seq, w.zipf_s)
                    sel = derive_selection(sc, n, V, w.alpha)
                    self.tables.append(_table(np.random.default_rng(w.seed * 1000 + version),
                                              version, dom_version, [sel], n, d))
                    self.domain_corpus.append(sc)
                    self.leaf_versions.append(version)
                    version += 1
            else:
                self.domain_corpus.append(corpus)
                self.leaf_versions.append(dom_version)
        self.n_leaves = len(self.leaf_versions)

    def tenant_version(self, t: int) -> int:
        return self.leaf_versions[t % self.n_leaves]

    def requests(self, seed: int, n: int, tenants=None):
        """n requests: (instance/tenant ids, tokens [n, seq], lens [n])."""
        w = self.w
        rng = np.random.default_rng(seed)
        pool = np.arange(w.n_tenants) if tenants is None else np.asarray(tenants)
        inst = pool[rng.integers(0, len(pool), n)].astype(np.uint32)
        toks = np.zeros((n, w.seq), np.uint32)
        for i, t in enumerate(inst):
            corpus = self.domain_corpus[int(t) % self.n_leaves].reshape(-1)
            off = int(rng.integers(0, corpus.size - w.seq + 1))
            toks[i] = corpus[off:off + w.seq]
        noise = rng.random((n, w.seq)) < w.p_noise
        toks[noise] = rng.integers(0, w.vocab_size, int(noise.sum()))
        lens = np.full(n, w.seq, np.uint32)
        return inst, toks, lens

    def table_rows(self) -> int:
        return int(sum(t["reps"].shape[0] for t in self.tables))
