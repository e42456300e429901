# SPDX-License-Identifier: Apache-2.0
"""Serving-side mirror of the reference's scheduler types over the CUDA backend.

Reference (proj/include/hmi/scheduler/request.hpp, SPEC.md scheduler module):

* ``InferRequest`` / ``InferBatch`` / ``InferResult``   request.hpp:15-44
* ``InstanceBinding`` / ``InstanceTable``               request.hpp:30-36
* ``BatchQueue`` — a request joins the last open batch; when that batch is
  full a new one is opened first; batch ids are sequential   request.hpp:48-64,
  SPEC.md:431-439 (9 requests at max 3 -> (3,3,3); 7 -> (3,3,1)).
* ``HeadOutput``                                        model.hpp:40-47

String ids (task_id, instance_id) are mapped to the dense indices the C ABI
uses. ``ShardRouter`` implements the multi-GPU placement of SURVEY.md §8(e):
tenant index mod world size, no collectives on the data path.
"""
from __future__ import annotations

import threading
import time
from collections import deque
from dataclasses import dataclass, field

import numpy as np

from ._native import ConflictError, RoutingError


@dataclass
class InferRequest:
    request_id: str
    tenant_id: str
    instance_id: str
    tokens: list
    enqueue_time_ms: float = 0.0


@dataclass
class InferBatch:
    batch_id: int
    requests: list = field(default_factory=list)


@dataclass
class InstanceBinding:
    version_id: int
    task_id: str
    head: str  # head id (the reference stores the OutputHead by value; dedup by id here)


@dataclass
class HeadOutput:
    kind: int = 0
    label: int = -1
    scores: list = field(default_factory=list)
    tags: list = field(default_factory=list)


@dataclass
class InferResult:
    request_id: str
    batch_id: int
    output: HeadOutput
    queue_ms: float = 0.0
    total_ms: float = 0.0


class BatchQueue:
    """request.hpp:48-64 with the SPEC's batching rule."""

    def __init__(self, max_batch_size: int):
        if max_batch_size < 1:
            raise ValueError("max_batch_size must be >= 1")
        self._max = max_batch_size
        self._next_id = 0
        self._batches: deque[InferBatch] = deque()
        self._mu = threading.Lock()

    @property
    def max_batch_size(self) -> int:
        return self._max

    def enqueue(self, req: InferRequest) -> int:
        with self._mu:
            if not self._batches or len(self._batches[-1].requests) >= self._max:
                self._batches.append(InferBatch(self._next_id))
                self._next_id += 1
            self._batches[-1].requests.append(req)
            return self._batches[-1].batch_id

    def take_all(self) -> list[InferBatch]:
        with self._mu:
            out = list(self._batches)
            self._batches.clear()
            return out

    def pending_requests(self) -> int:
        with self._mu:
            return sum(len(b.requests) for b in self._batches)

    def pending_batches(self) -> int:
        with self._mu:
            return len(self._batches)


class Registry:
    """String ids -> dense indices, and the InstanceTable."""

    def __init__(self):
        self.tasks: dict[str, int] = {}
        self.heads: dict[str, int] = {}
        self.instances: dict[str, int] = {}
        self.bindings: dict[str, InstanceBinding] = {}

    def task_index(self, task_id: str, create: bool = False) -> int:
        if task_id in self.tasks:
            if create:
                raise ConflictError(f"adapter set for task {task_id} already registered")
            return self.tasks[task_id]
        if not create:
            raise RoutingError(f"no adapter set registered for task {task_id}")
        self.tasks[task_id] = len(self.tasks)
        return self.tasks[task_id]

    def head_index(self, head_id: str, create: bool = False) -> int:
        if head_id not in self.heads:
            if not create:
                raise RoutingError(f"no output head {head_id}")
            self.heads[head_id] = len(self.heads)
        return self.heads[head_id]

    def bind(self, instance_id: str, binding: InstanceBinding) -> int:
        if instance_id in self.bindings:
            raise ConflictError(f"instance {instance_id} already bound")
        self.task_index(binding.task_id)
        self.head_index(binding.head)
        idx = self.instances.setdefault(instance_id, len(self.instances))
        self.bindings[instance_id] = binding
        return idx

    def instance_index(self, instance_id: str) -> int:
        if instance_id not in self.bindings:
            raise RoutingError(f"instance {instance_id} is not bound")
        return self.instances[instance_id]


class Server:
    """Drains a BatchQueue through one backend (GpuEngine or any object with the
    same ``infer_batch(instance_idx, tokens, lens)`` method), returning
    InferResults in batch order and request order."""

    def __init__(self, backend, registry: Registry, max_batch_size: int, max_seq: int,
                 head_kinds: dict[int, int] | None = None, manager=None):
        self.backend = backend
        self.registry = registry
        self.queue = BatchQueue(max_batch_size)
        self.max_seq = max_seq
        self.head_kinds = head_kinds or {}
        # manage.Manager: its queued mutations are applied between batches, never inside one
        self.manager = manager
        self.rejected: list[tuple[str, str]] = []  # (request_id, reason): queue conservation

    def enqueue(self, req: InferRequest) -> int:
        self.registry.instance_index(req.instance_id)  # unknown instance -> RoutingError
        if not req.tokens:
            raise ValueError("tokens must be non-empty")
        if req.enqueue_time_ms == 0.0:
            req.enqueue_time_ms = time.perf_counter() * 1e3
        return self.queue.enqueue(req)

    def run(self) -> list[InferResult]:
        results = []
        for batch in self.queue.take_all():
            if self.manager is not None:
                self.manager.apply_pending()
                kept = []
                for r in batch.requests:  # instances deleted since enqueue are rejected
                    if r.instance_id in self.registry.bindings:
                        kept.append(r)
                    else:
                        self.rejected.append((r.request_id, f"instance {r.instance_id} is not bound"))
                batch = InferBatch(batch.batch_id, kept)
                if not kept:
                    continue
            t_deq = time.perf_counter() * 1e3
            n = len(batch.requests)
            stride = max(len(r.tokens) for r in batch.requests)
            toks = np.zeros((n, stride), np.uint32)
            lens = np.zeros(n, np.uint32)
            inst = np.zeros(n, np.uint32)
            for i, r in enumerate(batch.requests):
                toks[i, :len(r.tokens)] = r.tokens
                lens[i] = len(r.tokens)
                inst[i] = self.registry.instance_index(r.instance_id)
            out = self.backend.infer_batch(inst, toks, lens, want_tags=True)
            t_done = time.perf_counter() * 1e3
            for i, r in enumerate(batch.requests):
                head = self.registry.bindings[r.instance_id].head
                kind = self.head_kinds.get(self.registry.head_index(head), 0)
                ho = HeadOutput(kind=kind)
                if kind == 1:
                    ho.tags = [int(x) for x in out.tags[i, :lens[i]]]
                else:
                    ho.label = int(out.labels[i])
                    ho.scores = [float(x) for x in out.scores[i]]
                results.append(InferResult(r.request_id, batch.batch_id, ho,
                                           t_deq - r.enqueue_time_ms, t_done - r.enqueue_time_ms))
        return results


class ShardRouter:
    """Tenant sharding across GPUs: task index t is owned by
    rank t % world_size unless it was moved (peer rebalancing, §8(f) rank 3).
    split() keeps arrival order within each shard; merge() restores the
    original order."""

    def __init__(self, world_size: int):
        self.world_size = world_size
        self.moved: dict[int, int] = {}

    def owner(self, task_idx: int) -> int:
        t = int(task_idx)
        return self.moved.get(t, t % self.world_size)

    def owners(self, task_of_request) -> np.ndarray:
        t = np.asarray(task_of_request).astype(np.int64)
        o = t % self.world_size
        if self.moved:
            keys = np.fromiter(self.moved.keys(), np.int64, len(self.moved))
            vals = np.fromiter(self.moved.values(), np.int64, len(self.moved))
            order = np.argsort(keys)
            keys, vals = keys[order], vals[order]
            pos = np.minimum(np.searchsorted(keys, t), len(keys) - 1)
            hit = keys[pos] == t
            o[hit] = vals[pos[hit]]
        return o

    def split(self, task_of_request) -> list[np.ndarray]:
        o = self.owners(task_of_request)
        return [np.nonzero(o == r)[0] for r in range(self.world_size)]

    def move(self, task_idx: int, rank: int) -> None:
        if not 0 <= rank < self.world_size:
            raise ValueError(f"rank {rank} outside [0, {self.world_size})")
        t = int(task_idx)
        if rank == t % self.world_size:
            self.moved.pop(t, None)
        else:
            self.moved[t] = int(rank)

    def plan_rebalance(self, load, tolerance: float = 0.1, max_moves: int = 64):
        """Greedy migration plan from per-task load (requests per task index over a window,
        identical on every rank, e.g. all-reduced): while the busiest rank exceeds the idlest by
        more than ``tolerance`` x the mean rank load, move the busiest rank's heaviest task whose
        load is at most half the gap (so the move never overshoots). Deterministic: ties break on
        the lower task index. Returns [(task, src_rank, dst_rank)]; apply with move() once the
        adapters have been migrated (GpuEngine.migrate_task / export_task + import_task)."""
        load = np.asarray(load, np.float64)
        tasks = np.nonzero(load > 0)[0]
        owner = {int(t): self.owner(int(t)) for t in tasks}
        rank_load = np.zeros(self.world_size)
        for t in tasks:
            rank_load[owner[int(t)]] += load[t]
        mean = rank_load.sum() / self.world_size
        plan = []
        while len(plan) < max_moves and mean > 0:
            hi = int(np.argmax(rank_load))
            lo = int(np.argmin(rank_load))
            gap = rank_load[hi] - rank_load[lo]
            if gap <= tolerance * mean:
                break
            cand = [(-load[t], int(t)) for t in tasks if owner[int(t)] == hi and load[t] <= gap / 2]
            if not cand:
                break
            _, t = min(cand)
            owner[t] = lo
            rank_load[hi] -= load[t]
            rank_load[lo] += load[t]
            plan.append((t, hi, lo))
        return plan

    def merge(self, parts: list[np.ndarray], values: list[np.ndarray], n: int):
        first = next(v for v in values if len(v))
        out = np.zeros((n,) + first.shape[1:], first.dtype)
        for idx, v in zip(parts, values):
            out[idx] = v
        return out
