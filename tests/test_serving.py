# SPDX-License-Identifier: Apache-2.0
"""Host-side serving logic: BatchQueue KATs, registry errors, tenant sharding.

The multi-process test runs world_size 2 over gloo on CPU: each rank serves
only its own tenants (t % 2 == rank) through a CPU backend built on the
oracle, and the merged per-request results equal the single-process run
exactly (sharding never changes per-request arithmetic)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2504_17449_b200._native import ConflictError, RoutingError
from paper_2504_17449_b200.engine import BatchResult
from paper_2504_17449_b200.serving import (BatchQueue, InferRequest, InstanceBinding, Registry,
                                           Server, ShardRouter)
from tests.world import World

CFG = oracle.Config(128, 2, 2, 2, 256, 300, 0, 3, 5)


def _req(i, inst="i0"):
    return InferRequest(f"r{i}", "t", inst, [1, 2, 3])


def test_batchqueue_spec_examples():
    """9 requests at max 3 -> (3,3,3); 7 -> (3,3,1); ids sequential."""
    q = BatchQueue(3)
    for i in range(9):
        q.enqueue(_req(i))
    b = q.take_all()
    assert [len(x.requests) for x in b] == [3, 3, 3] and [x.batch_id for x in b] == [0, 1, 2]
    for i in range(7):
        q.enqueue(_req(i))
    assert q.pending_batches() == 3 and q.pending_requests() == 7
    b = q.take_all()
    assert [len(x.requests) for x in b] == [3, 3, 1] and [x.batch_id for x in b] == [3, 4, 5]
    assert [r.request_id for r in b[0].requests] == ["r0", "r1", "r2"]  # arrival order


def test_registry_errors():
    r = Registry()
    r.task_index("a", create=True)
    with pytest.raises(ConflictError):
        r.task_index("a", create=True)
    r.head_index("h", create=True)
    r.bind("i1", InstanceBinding(0, "a", "h"))
    with pytest.raises(ConflictError):
        r.bind("i1", InstanceBinding(0, "a", "h"))
    with pytest.raises(RoutingError):
        r.bind("i2", InstanceBinding(0, "missing", "h"))
    with pytest.raises(RoutingError):
        r.instance_index("nope")


def test_shard_router_split_merge():
    rt = ShardRouter(4)
    tasks = np.array([5, 2, 8, 3, 0, 7, 6, 1])
    parts = rt.split(tasks)
    assert [list(p) for p in parts] == [[2, 4], [0, 7], [1, 6], [3, 5]]
    vals = [tasks[p] * 10 for p in parts]
    assert np.array_equal(rt.merge(parts, vals, len(tasks)), tasks * 10)


class OracleBackend:
    """CPU stand-in for GpuEngine (tests only): same infer_batch signature."""

    def __init__(self, world: World):
        self.w = world

    def infer_batch(self, inst, toks, lens, want_tags=False, want_trace=False):
        s, l, _ = self.w.oracle_batch(inst, toks, lens, threads=4)
        return BatchResult(s.astype(np.float32), l.astype(np.int32), None)


def test_server_bypass_oracle_cpu():
    """SPEC.md:540 / acceptance #11: a served request equals the direct
    higher_stack_forward(retrieve_sequence(tokens)) (CPU backend, bit-for-bit)."""
    w = World(CFG, n_tasks=4, r=8, labels=5, engine=False)
    reg = Registry()
    for t in range(4):
        reg.task_index(f"task{t}", create=True)
        reg.head_index(f"head{t}", create=True)
        reg.bind(f"inst{t}", InstanceBinding(int(w.inst_version[t]), f"task{t}", f"head{t}"))
    srv = Server(OracleBackend(w), reg, max_batch_size=3, max_seq=32)
    inst, toks, lens = w.requests(1, 5, 20)
    for i in range(5):
        srv.enqueue(InferRequest(f"r{i}", "tenant", f"inst{inst[i]}", list(toks[i, :lens[i]])))
    res = srv.run()
    assert [r.batch_id for r in res] == [0, 0, 0, 1, 1]
    for i, r in enumerate(res):
        s, lab, _ = w.oracle_one(int(inst[i]), toks[i], int(lens[i]))
        assert r.output.label == lab
        assert np.array_equal(np.float32(r.output.scores), s.astype(np.float32))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _shard_worker(rank, world_size, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world_size)
    w = World(CFG, n_tasks=6, r=8, labels=5, engine=False)
    inst, toks, lens = w.requests(9, 12, 24)
    router = ShardRouter(world_size)
    parts = router.split(inst)  # tenant index == instance index here
    mine = parts[rank]
    be = OracleBackend(w)
    res = be.infer_batch(inst[mine], toks[mine], lens[mine]) if len(mine) else None
    gathered = [None] * world_size
    dist.all_gather_object(gathered, (res.scores if res else np.zeros((0, 5), np.float32),
                                      res.labels if res else np.zeros(0, np.int32)))
    if rank == 0:
        scores = router.merge(parts, [g[0] for g in gathered], len(inst))
        labels = router.merge(parts, [g[1] for g in gathered], len(inst))
        ref = be.infer_batch(inst, toks, lens)
        out.put((np.array_equal(scores, ref.scores), np.array_equal(labels, ref.labels)))
    dist.barrier()
    dist.destroy_process_group()


def test_tenant_sharding_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shard_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    ok = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
    assert ok == (True, True)
