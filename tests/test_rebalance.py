# SPDX-License-Identifier: Apache-2.0
"""Peer rebalancing of tenants' adapters between engines.

CPU: the shard router's moves and its deterministic rebalance plan, agreed on by two gloo ranks
from all-reduced per-task load, leave every request's result unchanged (sharding never changes
per-row arithmetic, §8(e)). GPU: a task migrated (or replicated) device to device serves exactly
what it served before, including after eviction and refill from the host copy the import rebuilt
from HBM, within a process (peer copy) and across processes (CUDA IPC)."""
import ctypes
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2504_17449_b200 import _native
from paper_2504_17449_b200._native import ConfigError, ConflictError, RoutingError
from paper_2504_17449_b200.serving import ShardRouter
from tests.test_serving import CFG, OracleBackend, _free_port
from tests.world import World


def test_task_export_layout():
    # int32 device, int32 pid, u64 arena, u8[64] ipc handle, u64 slot_bytes, u64 fingerprint,
    # u32 layers, u32 task_idx, int32 slot[64]
    assert ctypes.sizeof(_native.TaskExport) == 4 + 4 + 8 + 64 + 8 + 8 + 4 + 4 + 4 * 64


def test_router_moves():
    rt = ShardRouter(4)
    tasks = np.array([5, 2, 8, 3, 0, 7, 6, 1, 5, 9])
    rt.move(5, 3)
    rt.move(2, 0)
    assert rt.owner(5) == 3 and rt.owner(2) == 0 and rt.owner(9) == 1
    assert list(rt.owners(tasks)) == [rt.owner(t) for t in tasks]
    parts = rt.split(tasks)
    assert [list(p) for p in parts] == [[1, 2, 4], [7, 9], [6], [0, 3, 5, 8]]
    rt.move(5, 1)  # back to its home rank: no longer an override
    assert 5 not in rt.moved and rt.owner(5) == 1
    with pytest.raises(ValueError):
        rt.move(3, 4)


def test_rebalance_plan():
    rt = ShardRouter(2)
    # rank 0 (even tasks) carries 3 hot tenants; rank 1 nearly idle
    load = np.zeros(12)
    load[[0, 2, 4]] = [50, 30, 20]
    load[[1, 3]] = [5, 5]
    plan = rt.plan_rebalance(load)
    assert plan == [(2, 0, 1)]
    for t, src, dst in plan:
        assert rt.owner(t) == src
        rt.move(t, dst)
    per = [sum(load[t] for t in range(12) if rt.owner(t) == r) for r in range(2)]
    assert abs(per[0] - per[1]) < 50  # the heaviest single tenant bounds the best split
    assert rt.plan_rebalance(load) == []  # balanced within tolerance: nothing more to move
    # a single tenant heavier than half the gap is never moved (it would overshoot)
    assert ShardRouter(2).plan_rebalance(np.array([100.0, 0.0])) == []
    # deterministic: same load, same plan
    assert ShardRouter(3).plan_rebalance(load) == ShardRouter(3).plan_rebalance(load.copy())


def _rebalance_worker(rank, world_size, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world_size)
    w = World(CFG, n_tasks=6, r=8, labels=5, engine=False)
    inst, toks, lens = w.requests(31, 14, 24)
    inst[:8] = np.array([0, 2, 4, 0, 2, 0, 4, 0], np.uint32)  # skew onto rank 0's tenants
    router = ShardRouter(world_size)
    # each rank counts the requests of the tenants it owns; the all-reduced vector is the same
    # everywhere, so every rank derives the same plan without a coordinator
    mine = router.split(inst)[rank]
    counts = torch.zeros(6, dtype=torch.float64)
    for t in inst[mine]:
        counts[int(t)] += 1
    dist.all_reduce(counts)
    plan = router.plan_rebalance(counts.numpy())
    plans = [None] * world_size
    dist.all_gather_object(plans, plan)
    for t, _, dst in plan:
        router.move(t, dst)
    parts = router.split(inst)
    be = OracleBackend(w)
    res = be.infer_batch(inst[parts[rank]], toks[parts[rank]], lens[parts[rank]])
    gathered = [None] * world_size
    dist.all_gather_object(gathered, (res.scores, res.labels))
    if rank == 0:
        scores = router.merge(parts, [g[0] for g in gathered], len(inst))
        labels = router.merge(parts, [g[1] for g in gathered], len(inst))
        ref = be.infer_batch(inst, toks, lens)
        sizes = [len(p) for p in parts]
        out.put((plans[0] == plans[1], len(plan) > 0, max(sizes) - min(sizes),
                 np.array_equal(scores, ref.scores), np.array_equal(labels, ref.labels)))
    dist.barrier()
    dist.destroy_process_group()


def test_rebalance_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rebalance_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    same_plan, moved, spread, eq_s, eq_l = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
    assert same_plan and moved and eq_s and eq_l
    assert spread <= 4


# ---------------------------------------------------------------------------------------- GPU
def _peer_engine(w: World, pool_bytes=0, r=None):
    """An engine with w's model, tables and heads but no tasks (they arrive by import)."""
    from paper_2504_17449_b200 import engine as E

    c = w.cfg
    mc = E.model_config(c.hidden_size, c.heads, c.lower_layers, c.higher_layers, c.ffn_size,
                        c.vocab_size, c.mode, c.max_fragment, c.seed)
    eng = E.GpuEngine(mc, w.higher, max_batch=32, max_seq=128, bottleneck=r or w.r,
                      max_labels=w.labels, pool_bytes=pool_bytes, max_tasks=len(w.adapters),
                      max_versions=max(8, w.n_versions))
    for t in w.tables:
        eng.upload_table(t["version"], t["parent"], t["key_len"], t["keys"], t["reps"])
    for t in range(len(w.adapters)):
        wh, b = w.heads[t]
        eng.register_head(t, w.head_kind, wh, b)
    return eng


def _bind(eng, w, t):
    eng.bind_instance(t, int(w.inst_version[t]), t, t)


@pytest.mark.gpu
def test_migrate_and_replicate_same_process():
    w = World(CFG, n_tasks=6, r=8, labels=5)
    inst, toks, lens = w.requests(41, 24, 40)
    inst = (inst % 3 + 1).astype(np.uint32)  # tasks 1, 2, 3
    sub = {t: np.nonzero(inst == t)[0] for t in (1, 2, 3)}
    before = w.eng.infer_batch(inst, toks, lens)
    c = CFG
    layer_bytes = (c.hidden_size * w.r * 2 + w.r + c.hidden_size) * 4
    # the destination's slot pool holds one task: serving the three in turn forces eviction and
    # refills from the host copy the import rebuilt from HBM
    b = _peer_engine(w, pool_bytes=c.higher_layers * layer_bytes)
    for t in (1, 2, 3):
        ex = _native.TaskExport.from_buffer_copy(w.eng.export_task(t))
        assert ex.layers == c.higher_layers and ex.task_idx == t
        assert all(ex.slot[l] >= 0 for l in range(ex.layers))
        w.eng.release_export(t)
        moved = w.eng.migrate_task(b, t, keep_source=(t == 3))
        assert moved == ex.slot_bytes * ex.layers
        _bind(b, w, t)
    loads0 = b.pool_stats()["loads"]
    for _ in range(2):
        for t, idx in sub.items():
            after = b.infer_batch(inst[idx], toks[idx], lens[idx])
            assert np.array_equal(after.scores, before.scores[idx]), t
            assert np.array_equal(after.labels, before.labels[idx]), t
    assert b.pool_stats()["loads"] > loads0  # refills from the rebuilt host copies happened
    # migrated tasks left the source; the replicated one still serves there, identically
    with pytest.raises(RoutingError):
        w.eng.infer_batch(np.array([1], np.uint32), toks[:1], lens[:1])
    again = w.eng.infer_batch(inst[sub[3]], toks[sub[3]], lens[sub[3]])
    assert np.array_equal(again.scores, before.scores[sub[3]])
    # errors: duplicate import, release without export, replace / unregister while exported,
    # mismatched bottleneck
    ex3 = w.eng.export_task(3)
    with pytest.raises(ConflictError):
        b.import_task(3, ex3)
    with pytest.raises(ConflictError):
        w.eng.unregister_task(3)
    with pytest.raises(ConflictError):
        w.eng.replace_task(3, w.adapters[3])
    other = _peer_engine(w, r=16)
    with pytest.raises(ConfigError):
        other.import_task(3, ex3)
    other.close()
    w.eng.release_export(3)
    with pytest.raises(RoutingError):
        w.eng.release_export(3)
    with pytest.raises(RoutingError):
        w.eng.export_task(1)  # no longer registered at the source
    # an import carrying the f32 adapter builds its host copy from it instead of from HBM
    ex0 = w.eng.export_task(0)
    b.import_task(0, ex0, adapter_f32=w.adapters[0])
    w.eng.release_export(0, drop=True)
    _bind(b, w, 0)
    sel = np.array([0, 0, 0], np.uint32)
    got = b.infer_batch(sel, toks[:3], lens[:3])
    s, lab, _ = w.oracle_batch(sel, toks[:3], lens[:3], threads=4)
    from tests.world import logit_error
    assert logit_error(got.scores, s) <= 2e-2
    b.close()
    w.eng.close()


def _ipc_source(q_out, q_in):
    w = World(CFG, n_tasks=6, r=8, labels=5)
    q_out.put(w.eng.export_task(2))
    q_in.get(timeout=300)  # importer done
    w.eng.release_export(2, drop=True)
    w.eng.close()
    q_out.put("released")


@pytest.mark.gpu
def test_migrate_across_processes_ipc():
    ctx = mp.get_context("spawn")
    q_out, q_in = ctx.Queue(), ctx.Queue()
    p = ctx.Process(target=_ipc_source, args=(q_out, q_in))
    p.start()
    try:
        blob = q_out.get(timeout=300)
        w = World(CFG, n_tasks=6, r=8, labels=5)
        inst, toks, lens = w.requests(43, 8, 40)
        inst[:] = 2
        ref = w.eng.infer_batch(inst, toks, lens)
        b = _peer_engine(w)
        ex = _native.TaskExport.from_buffer_copy(blob)
        assert ex.pid != os.getpid()
        moved = b.import_task(2, blob)
        assert moved == ex.slot_bytes * ex.layers
        q_in.put("done")
        _bind(b, w, 2)
        got = b.infer_batch(inst, toks, lens)
        assert np.array_equal(got.scores, ref.scores)
        assert q_out.get(timeout=120) == "released"
        # the source process is gone; the imported task lives on in this engine's own slots
        again = b.infer_batch(inst, toks, lens)
        assert np.array_equal(again.scores, ref.scores)
        b.close()
        w.eng.close()
    finally:
        p.join(timeout=120)
        if p.is_alive():
            p.kill()
