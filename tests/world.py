# SPDX-License-Identifier: Apache-2.0
"""Shared fixture: one seeded multi-tenant "world" loaded into both the GPU
engine and the CPU oracle (identical weights, tables, adapters, heads)."""
from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor

import numpy as np

import oracle
from paper_2504_17449_b200 import engine as E
from tests.synth_tables import make_requests, make_tree

ADAPTER_SEED = 1000       # adapter seed = 1000 + tenant_idx
HEAD_SEED = 2_000_000     # head seed = 2e6 + tenant_idx


class World:
    def __init__(self, cfg: oracle.Config, n_tasks: int, r: int, labels: int, *,
                 head_kind: int = 0, branches=((0, 40), (0, 40), (1, 30)), max_batch=32,
                 max_seq=128, pool_bytes=0, pipeline_mode=E.MODE_FINE, precision=0,
                 table_seed=1, n_hot=24, n_bi=80, n_tri=60, engine=True, shared_head=False,
                 max_new_tokens=0, max_labels=None, tasks=None, device=0):
        self.cfg, self.r, self.labels, self.head_kind = cfg, r, labels, head_kind
        self.higher = oracle.generate_higher(cfg)
        self.tables, self.hot = make_tree(table_seed, cfg.vocab_size, cfg.hidden_size,
                                          cfg.max_fragment, n_hot=n_hot, n_bi=n_bi,
                                          n_tri=n_tri, branches=branches)
        self.tree = oracle.OracleTree(cfg.max_fragment, cfg.hidden_size)
        for t in self.tables:
            self.tree.add_table(t["version"], t["parent"], t["key_len"], t["keys"], t["reps"])
        self.adapters = [oracle.generate_adapter(cfg, r, ADAPTER_SEED + t) for t in range(n_tasks)]
        # shared_head: one (vocabulary-wide lm) head bound to every instance
        self.heads = [oracle.generate_head(cfg.hidden_size, labels, HEAD_SEED + (0 if shared_head else t))
                      for t in range(1 if shared_head else n_tasks)]
        self.shared_head = shared_head
        self.n_versions = len(self.tables)
        # instance i -> (version i % n_versions, task i, head i)
        self.inst_version = np.arange(n_tasks) % self.n_versions
        self.eng = None
        if engine:
            mc = E.model_config(cfg.hidden_size, cfg.heads, cfg.lower_layers, cfg.higher_layers,
                                cfg.ffn_size, cfg.vocab_size, cfg.mode, cfg.max_fragment,
                                cfg.seed)
            self.eng = E.GpuEngine(mc, self.higher, device=device, precision=precision,
                                   max_batch=max_batch,
                                   max_seq=max_seq, bottleneck=r,
                                   max_labels=labels if max_labels is None else max_labels,
                                   pipeline_mode=pipeline_mode, pool_bytes=pool_bytes,
                                   max_tasks=n_tasks, max_versions=max(8, self.n_versions),
                                   max_new_tokens=max_new_tokens)
            for t in self.tables:
                self.eng.upload_table(t["version"], t["parent"], t["key_len"], t["keys"], t["reps"])
            # tasks: the subset this engine serves (a tenant shard), default all
            for t in (range(n_tasks) if tasks is None else tasks):
                self.eng.register_task(t, self.adapters[t])
                if not shared_head or t == 0:
                    w, b = self.heads[t]
                    self.eng.register_head(t, head_kind, w, b)
                self.eng.bind_instance(t, int(self.inst_version[t]), t, 0 if shared_head else t)

    def requests(self, seed, n, max_len, min_len=1, p_hot=0.9):
        toks, lens = make_requests(seed, n, self.hot, self.cfg.vocab_size, max_len,
                                   min_len=min_len, p_hot=p_hot)
        inst = np.random.default_rng(seed + 99).integers(0, len(self.adapters), n)
        return inst.astype(np.uint32), toks, lens

    def oracle_one(self, inst, tokens, length):
        w, b = self.heads[0 if self.shared_head else inst]
        return oracle.infer_one(self.cfg, self.higher, self.tree, int(self.inst_version[inst]),
                                tokens[:length], self.adapters[inst], self.r, w, b,
                                head_kind=self.head_kind)

    def oracle_batch(self, inst, toks, lens, threads=16):
        with ThreadPoolExecutor(threads) as ex:
            res = list(ex.map(lambda i: self.oracle_one(int(inst[i]), toks[i], int(lens[i])),
                              range(len(inst))))
        scores = np.stack([r[0] for r in res])
        labels = np.array([r[1] for r in res])
        tags = [r[2] for r in res]
        return scores, labels, tags


def logit_error(gpu_scores, ref_scores):
    """max over requests of ||delta||_inf / ||ref||_inf."""
    L = ref_scores.shape[1]
    d = np.abs(gpu_scores[:, :L].astype(np.float64) - ref_scores).max(axis=1)
    return float((d / np.abs(ref_scores).max(axis=1)).max())


def token_tag_check(world, inst, toks, lens, gpu_tags, gpu_hidden):
    """Per-token argmax check of a token_tag batch (apply_head, model.cpp:158-163) with every
    disagreement classified. Reference rows: the oracle's final (post-LN2) rows of each request;
    GPU rows: the engine's normalised final rows (debug flag 2). For each row p < len, scores
    are rows @ W + b in f64; a mismatched tag is a near-tie when the reference's margin between
    its tag and the GPU's (relative to the row's max |score|) is within twice that row's
    measured score error, else decisive. Returns (agreement, n_tokens, decisive, near_ties)."""
    agree = total = 0
    decisive, ties = [], []
    for i in range(len(inst)):
        k, n = int(inst[i]), int(lens[i])
        w, b = world.heads[0 if world.shared_head else k]
        h0, _, _, _ = world.tree.retrieve(int(world.inst_version[k]), toks[i, :n], world.cfg.mode)
        _, _, tags, h = oracle.higher_forward(world.cfg, world.higher, h0, n, world.adapters[k],
                                              world.r, w, b, head_kind=1)
        W, B = np.asarray(w, np.float64), np.asarray(b, np.float64)
        ref_s = h[:n] @ W + B
        gpu_s = gpu_hidden[i, :n].astype(np.float64) @ W + B
        scale = np.abs(ref_s).max(axis=1)
        err = np.abs(gpu_s - ref_s).max(axis=1) / scale
        for p in range(n):
            total += 1
            g, r = int(gpu_tags[i, p]), int(tags[p])
            if g == r:
                agree += 1
                continue
            m = float((ref_s[p, r] - ref_s[p, g]) / scale[p])
            (ties if m <= 2 * err[p] else decisive).append((i, p, m, float(err[p])))
    return agree / max(total, 1), total, decisive, ties
