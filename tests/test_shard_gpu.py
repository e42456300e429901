# SPDX-License-Identifier: Apache-2.0
"""Tenant sharding through the product path: two ranks (gloo, sharing the
one GPU of this box), each owning a GpuEngine that registers only its own tenants
(t % 2 == rank, ShardRouter) with its own HBM slot pool sized for about half of them, so
adapters swap in and out. A stream of mixed-tenant batches is split by owner, each rank
serves its share, results are all-gathered and merged back into arrival order; rank 0
checks the merged scores and labels bit for bit against ONE engine holding every
tenant, and the labels against the CPU oracle. No collective touches the data path: the
exchange here is the test's own result gathering."""
import datetime
import os
import socket
import traceback

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2504_17449_b200 import engine as E
from paper_2504_17449_b200.serving import ShardRouter
from tests.world import World

pytestmark = pytest.mark.gpu

N_TASKS, R, LABELS = 24, 16, 6
BATCHES = [(31 + k, 20, 128) for k in range(4)]  # (seed, requests, max length)


def _world(**kw):
    return World(oracle.TINY, n_tasks=N_TASKS, r=R, labels=LABELS, max_batch=32, **kw)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _layer_bytes():
    d = oracle.TINY.hidden_size
    return (d * R * 2 + R + d) * 4 * oracle.TINY.higher_layers


def _worker(rank, world_size, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world_size,
                            timeout=datetime.timedelta(seconds=300))
    try:
        router = ShardRouter(world_size)
        mine = [t for t in range(N_TASKS) if router.owner(t) == rank]
        probe = _world(engine=False)
        reqs = [probe.requests(*b) for b in BATCHES]
        worst = max(len(set(inst[router.split(inst)[rank]].tolist())) for inst, _, _ in reqs)
        pool_tasks = max(worst, len(mine) // 2)
        w = _world(tasks=mine, pool_bytes=pool_tasks * _layer_bytes())
        out = []
        for inst, toks, lens in reqs:
            part = router.split(inst)[rank]
            res = w.eng.infer_batch(inst[part], toks[part], lens[part], want_tags=True) if len(part) else None
            out.append((part, None if res is None else (res.scores, res.labels)))
        stats = w.eng.pool_stats()
        numa = E.engine_counters(w.eng)["numa_node"]
        w.eng.close()
        gathered = [None] * world_size
        dist.all_gather_object(gathered, (out, stats, numa))
        if rank == 0:
            single = _world()
            ok_scores, ok_labels, ok_oracle, n = True, True, True, 0
            for k, (inst, toks, lens) in enumerate(reqs):
                parts = [g[0][k][0] for g in gathered]
                vals = [g[0][k][1] for g in gathered]
                scores = router.merge(parts, [v[0] if v is not None else np.zeros((0, LABELS), np.float32)
                                              for v in vals], len(inst))
                labels = router.merge(parts, [v[1] if v is not None else np.zeros(0, np.int32)
                                              for v in vals], len(inst))
                ref = single.eng.infer_batch(inst, toks, lens)
                ok_scores &= bool(np.array_equal(scores, ref.scores))
                ok_labels &= bool(np.array_equal(labels, ref.labels))
                _, ol, _ = single.oracle_batch(inst, toks, lens, threads=8)
                ok_oracle &= bool(np.mean(ol == labels) >= 0.999)
                n += len(inst)
            single.eng.close()
            q.put({"scores_bit_identical": ok_scores, "labels_bit_identical": ok_labels,
                   "labels_match_oracle": ok_oracle, "requests": n,
                   "loads": [g[1]["loads"] for g in gathered],
                   "capacity_tasks": [g[1]["capacity_bytes"] // _layer_bytes() for g in gathered],
                   "numa": [g[2] for g in gathered]})
        dist.barrier()
    except Exception:
        q.put({"error": f"rank {rank}: {traceback.format_exc()}"})
        raise
    finally:
        dist.destroy_process_group()


def test_two_rank_tenant_shards_match_one_engine():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    try:
        rec = q.get(timeout=600)
    finally:
        for p in procs:
            p.join(timeout=120)
    print(rec)
    assert "error" not in rec, rec["error"]
    assert rec["scores_bit_identical"] and rec["labels_bit_identical"], rec
    assert rec["labels_match_oracle"], rec
    # each shard's pool held about half its tenants, so the stream swapped adapters
    assert all(c < N_TASKS // 2 for c in rec["capacity_tasks"]), rec
    L = oracle.TINY.higher_layers  # loads count (task, layer) slots
    assert all(l > c * L for l, c in zip(rec["loads"], rec["capacity_tasks"])), rec
    assert all(p.exitcode == 0 for p in procs)
