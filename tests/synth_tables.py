# SPDX-License-Identifier: Apache-2.0
"""Small seeded PLOT trees + request streams for the parity tests.

Tables are synthetic seeded f32 rows (SPEC.md:676 allows synthetic tables);
keys are drawn from a small "hot" token set so requests exercise every
resolution level: whole-window hits, bi-gram fallback, uni-gram backstop,
branch shadowing of root keys, and parent-chain walks.
"""
from __future__ import annotations

import numpy as np


def _unique_keys(rng, hot, k, count, exclude=()):
    seen = set(exclude)
    out = []
    tries = 0
    while len(out) < count and tries < count * 50:
        tries += 1
        key = tuple(int(x) for x in rng.choice(hot, k))
        if key in seen:
            continue
        seen.add(key)
        out.append(key)
    return out


def make_tree(seed: int, vocab: int, d: int, ngram: int = 3, n_hot: int = 24,
              n_bi: int = 80, n_tri: int = 60, branches=((0, 40), (0, 40), (1, 30))):
    """Returns (tables, hot) where tables is a list of dicts in upload order:
    {version, parent, key_len[n], keys[n, ngram], reps[rows, d]}; version 0 is
    the root (parent 0xffffffff). `branches` = (parent_version, n_trigrams)."""
    rng = np.random.default_rng(seed)
    hot = rng.choice(vocab, n_hot, replace=False)
    keys = [(t,) for t in range(vocab)]  # uni-gram backstop (table.cpp:51-56)
    if ngram >= 2:
        keys += _unique_keys(rng, hot, 2, n_bi)
    if ngram >= 3:
        keys += _unique_keys(rng, hot, 3, n_tri)
    tables = [_table(rng, 0, 0xFFFFFFFF, keys, ngram, d)]
    root_tri = [k for k in keys if len(k) == ngram]
    for i, (parent, n) in enumerate(branches):
        # half shadow existing root keys, half are new
        shadow = [root_tri[j] for j in rng.choice(len(root_tri), min(n // 2, len(root_tri)),
                                                  replace=False)] if root_tri else []
        fresh = _unique_keys(rng, hot, ngram, n - len(shadow), exclude=shadow)
        tables.append(_table(rng, i + 1, parent, shadow + fresh, ngram, d))
    return tables, hot


def _table(rng, version, parent, keys, ngram, d):
    keys = sorted(set(keys))  # std::map order (PLT1 order, plot_io.cpp:26)
    key_len = np.array([len(k) for k in keys], np.uint32)
    karr = np.zeros((len(keys), ngram), np.uint32)
    for i, k in enumerate(keys):
        karr[i, :len(k)] = k
    rows = int(key_len.sum())
    reps = rng.standard_normal((rows, d)).astype(np.float32)
    return {"version": version, "parent": parent, "key_len": key_len, "keys": karr, "reps": reps}


def make_requests(seed: int, n: int, hot, vocab: int, max_len: int, min_len: int = 1,
                  p_hot: float = 0.9):
    rng = np.random.default_rng(seed)
    lens = rng.integers(min_len, max_len + 1, n).astype(np.uint32)
    toks = np.zeros((n, max_len), np.uint32)
    for i in range(n):
        L = lens[i]
        hotpick = rng.random(L) < p_hot
        toks[i, :L] = np.where(hotpick, rng.choice(hot, L), rng.integers(0, vocab, L))
    return toks, lens
