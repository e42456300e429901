# SPDX-License-Identifier: Apache-2.0
"""Physical slot placement of the product's SlotPool (CPU, host-only C ABI).

The engine sizes its HBM adapter pool as floor(n/L)*L + L*max_batch physical slots in blocks of
L = n_layers and places a task's layer l at slot block*L + l of the block the task claims, so a
whole-task load is one contiguous copy (engine.cpp, slot_pool.cpp take_slot). Placement must
never change a residency decision: the LoadRecords of a placed pool equal the accounting-only
pool's (whose law test_pool_parity.py pins to the reference DeviceSlotPool,
proj/src/adapters/device_pool.cpp), every resident layer owns a distinct in-range slot, and a
task loaded whole while a block was free sits in one block.
"""
import ctypes

import numpy as np
import pytest

from paper_2504_17449_b200 import _native
from paper_2504_17449_b200._native import check
from paper_2504_17449_b200.engine import SlotPoolPolicy

L = 4                 # layers per task = block length
LAYER_BYTES = 1000
N_TASKS = 40


def _pools(cap_tasks, max_batch):
    cap = cap_tasks * L * LAYER_BYTES
    slots = cap_tasks * L + L * max_batch  # engine.cpp pool sizing
    placed = SlotPoolPolicy(cap, physical_slots=slots, block_len=L)
    plain = SlotPoolPolicy(cap)
    for t in range(N_TASKS):
        placed.register(t, L, LAYER_BYTES)
        plain.register(t, L, LAYER_BYTES)
    return placed, plain, slots


def _check_slots(pool, slots):
    seen = {}
    for t in range(N_TASKS):
        for l in range(L):
            s = pool.slot(t, l)
            if s < 0:
                continue
            assert 0 <= s < slots, (t, l, s)
            assert s not in seen, f"slot {s} shared by {seen[s]} and {(t, l)}"
            seen[s] = (t, l)
    return seen


@pytest.mark.parametrize("seed", range(6))
def test_placement_keeps_decisions_and_slots_distinct(seed):
    rng = np.random.default_rng(seed)
    max_batch = 6
    placed, plain, slots = _pools(cap_tasks=10, max_batch=max_batch)
    pinned = []
    for _ in range(300):
        batch = sorted(set(rng.integers(0, N_TASKS, rng.integers(1, max_batch + 1)).tolist()))
        kind = rng.integers(0, 4)
        if kind == 0:  # fine mode: the per-layer calls of one batch, pinned across the batch
            placed.pin(batch)
            plain.pin(batch)
            for layer in range(L):
                a = placed.try_ensure_layer_resident(batch, layer)
                b = plain.try_ensure_layer_resident(batch, layer)
                assert a == b
                _check_slots(placed, slots)
            placed.unpin(batch)
            plain.unpin(batch)
        elif kind == 1:
            try:
                a = placed.ensure_resident(batch)
            except Exception as e:
                a = ("error", getattr(e, "code", -1))
            try:
                b = plain.ensure_resident(batch)
            except Exception as e:
                b = ("error", getattr(e, "code", -1))
            assert a == b
        elif kind == 2 and len(pinned) < 2:
            placed.pin(batch)
            plain.pin(batch)
            pinned.append(batch)
        elif kind == 3 and pinned:
            pb = pinned.pop(0)
            placed.unpin(pb)
            plain.unpin(pb)
        else:
            t = int(rng.integers(0, N_TASKS))
            assert placed.evict(t) == plain.evict(t)
        _check_slots(placed, slots)
        sa, sb = placed.stats(), plain.stats()
        assert sa == sb


def test_whole_task_loads_fill_one_block():
    placed, _, slots = _pools(cap_tasks=8, max_batch=4)
    for t in range(8):  # fits: every task claims a free block
        placed.ensure_resident([t])
        s = [placed.slot(t, l) for l in range(L)]
        assert s[0] % L == 0 and s == list(range(s[0], s[0] + L)), (t, s)
    # evictions free whole blocks again: the next whole-task loads stay contiguous
    for t in range(8, 20):
        placed.ensure_resident([t])
        s = [placed.slot(t, l) for l in range(L)]
        assert s[0] % L == 0 and s == list(range(s[0], s[0] + L)), (t, s)
    _check_slots(placed, slots)


def test_fine_mode_layers_land_in_the_claimed_block():
    placed, _, slots = _pools(cap_tasks=8, max_batch=4)
    batch = [3, 7, 11]
    placed.pin(batch)
    for layer in range(L):
        placed.try_ensure_layer_resident(batch, layer)
    for t in batch:
        s = [placed.slot(t, l) for l in range(L)]
        assert all(x >= 0 for x in s)
        assert s == list(range(s[0], s[0] + L)) and s[0] % L == 0, (t, s)
    placed.unpin(batch)
    assert placed.slot(0, 0) == -1  # never loaded
    _check_slots(placed, slots)


def test_placed_pool_rejects_zero_slots():
    h = ctypes.c_void_p()
    with pytest.raises(Exception):
        check(_native.lib().hmi_pool_create_placed(1000, 0, 4, ctypes.byref(h)))
