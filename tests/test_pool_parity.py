# SPDX-License-Identifier: Apache-2.0
"""Swap-trace parity: the product's slot-pool policy vs the reference DeviceSlotPool.

The same access trace is replayed through the reference (oracle/_ref, compiled
from proj/src/adapters/device_pool.cpp) and through the product's SlotPool
(paper_2504_17449_b200/csrc/slot_pool.cpp, via the host-only C ABI
hmi_pool_*). LoadRecords (hit, bytes, evicted) must match exactly.
Runs on CPU: no GPU is involved in residency decisions.
"""
import ctypes

import numpy as np
import pytest

import oracle
from paper_2504_17449_b200.engine import SlotPoolPolicy

D, R, LAYERS = 32, 8, 3
LAYER_BYTES = (D * R * 2 + R + D) * 4  # adapter_set.hpp:24-27 (f32 accounting)


class RefPool:
    def __init__(self, capacity):
        self.L = oracle.ref()
        if self.L is None:
            pytest.skip("reference library unavailable")
        self.h = self.L.ref_pool_create(capacity)

    def __del__(self):
        if getattr(self, "h", None):
            self.L.ref_pool_free(self.h)

    def register(self, task):
        assert self.L.ref_pool_register(self.h, f"t{task:05d}".encode(), LAYERS, D, R) == 0

    def op(self, op, tasks, layer=0):
        n = len(tasks)
        ids = (ctypes.c_char_p * max(n, 1))(*[f"t{t:05d}".encode() for t in tasks])
        hit = np.zeros(max(n, 1), np.int32)
        by = np.zeros(max(n, 1), np.uint64)
        ev = ctypes.create_string_buffer(1 << 16)
        k = self.L.ref_pool_op(self.h, op, n, ids, layer, oracle.ptr(hit, oracle.i32p),
                               oracle.ptr(by, oracle.u64p), ev, 1 << 16)
        if op == 1 and k == -1:
            return None
        if k < -1:
            return ("error", -k)
        if op >= 2:
            return int(k)
        evs = ev.value.decode().split(";")[:-1]
        return [{"hit": bool(hit[i]), "bytes": int(by[i]),
                 "evicted": [int(x[1:]) for x in evs[i].split(",") if x]} for i in range(k)]

    def stats(self):
        o = np.zeros(5, np.uint64)
        self.L.ref_pool_stats(self.h, oracle.ptr(o, oracle.u64p))
        return dict(zip(("hits", "loads", "resident_bytes", "max_resident_bytes_seen",
                         "resident_task_count"), map(int, o)))


def _ours(pool, op, tasks, layer=0):
    try:
        out = pool.op(op, tasks, layer)
    except Exception as e:  # map to the reference's status
        return ("error", getattr(e, "code", -1))
    if isinstance(out, list):
        return [{"hit": r["hit"], "bytes": r["bytes"], "evicted": r["evicted"]} for r in out]
    return out


def test_spec_lru_example():
    """capacity 2 sets, accesses A,B,A,C -> C evicts B, A stays."""
    cap = 2 * LAYERS * LAYER_BYTES
    ours, ref = SlotPoolPolicy(cap), RefPool(cap)
    for t in (0, 1, 2):
        ours.register(t, LAYERS, LAYER_BYTES)
        ref.register(t)
    for t in (0, 1, 0, 2):
        a, b = _ours(ours, 0, [t]), ref.op(0, [t])
        assert a == b
    assert b[0]["evicted"] == [1]


@pytest.mark.parametrize("seed", range(6))
def test_random_trace_parity(seed):
    rng = np.random.default_rng(seed)
    n_tasks = 40
    cap = int(rng.integers(3, 12)) * LAYER_BYTES + int(rng.integers(0, LAYER_BYTES))
    ours, ref = SlotPoolPolicy(cap), RefPool(cap)
    for t in range(n_tasks):
        ours.register(t, LAYERS, LAYER_BYTES)
        ref.register(t)
    pinned = []
    for step in range(400):
        kind = rng.random()
        batch = [int(x) for x in rng.integers(0, n_tasks, int(rng.integers(1, 5)))]
        if kind < 0.45:
            layer = int(rng.integers(0, LAYERS))
            a = _ours(ours, 1, batch, layer)
            b = ref.op(1, batch, layer)
        elif kind < 0.7:
            a, b = _ours(ours, 0, batch), ref.op(0, batch)
        elif kind < 0.8:
            a, b = _ours(ours, 2, batch), ref.op(2, batch)
            pinned.append(batch)
        elif kind < 0.9 and pinned:
            pb = pinned.pop(0)
            a, b = _ours(ours, 3, pb), ref.op(3, pb)
        elif kind < 0.95:
            a, b = _ours(ours, 4, batch), ref.op(4, batch)
        else:
            a, b = _ours(ours, 5, batch[:1]), ref.op(5, batch[:1])
        assert a == b, (step, kind, batch, a, b)
        assert ours.stats()["resident_bytes"] <= cap
    s1, s2 = ours.stats(), ref.stats()
    for k in s2:
        assert s1[k] == s2[k], k


def test_capacity_error_single_set_too_large():
    ours, ref = SlotPoolPolicy(LAYER_BYTES * 2), RefPool(LAYER_BYTES * 2)
    ours.register(0, LAYERS, LAYER_BYTES)
    ref.register(0)
    assert _ours(ours, 0, [0]) == ("error", 4) == ref.op(0, [0])
