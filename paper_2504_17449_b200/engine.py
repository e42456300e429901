# SPDX-License-Identifier: Apache-2.0
"""Host-side mirror of the reference serving API over the CUDA backend.

The reference's registration / serving types (proj/include/hmi/...):

=============================  =============================================
reference                      here
=============================  =============================================
ModelConfig (config.hpp)       :class:`ModelConfig` (ctypes struct)
ModelArtifacts.higher          ``higher_f32`` passed to :class:`GpuEngine`
VersionTree::add_branch        :meth:`GpuEngine.upload_table`
AdapterStore::register_set     :meth:`GpuEngine.register_task`
OutputHead                     :meth:`GpuEngine.register_head`
InstanceBinding / bind         :meth:`GpuEngine.bind_instance`
stage_compute + head           :meth:`GpuEngine.infer_batch`
DeviceSlotPool counters        :meth:`GpuEngine.pool_stats`
=============================  =============================================

String ids (tenant / instance / task) map to dense indices in
:mod:`paper_2504_17449_b200.serving`; this module speaks indices only, like
the C ABI (include/hmi_gpu.h).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _native
from ._native import LoadRecord, ModelConfig, Options, check

P = ctypes.POINTER
NO_PARENT = 0xFFFFFFFF

MODE_SYNC, MODE_COARSE, MODE_FINE = 0, 1, 2
HEAD_CLS, HEAD_TAG, HEAD_LM = 0, 1, 2


def _p(a, t):
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(P(t))


def model_config(hidden_size, heads, lower_layers, higher_layers, ffn_size, vocab_size,
                 mode=0, max_fragment=3, seed=7) -> ModelConfig:
    return ModelConfig(hidden_size, heads, lower_layers, higher_layers, ffn_size, vocab_size,
                       mode, max_fragment, seed)


def layer_floats(cfg: ModelConfig) -> int:
    d, f = cfg.hidden_size, cfg.ffn_size
    return 4 * (d * d + d) + (d * f + f) + (f * d + d) + 4 * d


def adapter_layer_floats(cfg: ModelConfig, r: int) -> int:
    d = cfg.hidden_size
    return d * r + r + r * d + d


@dataclass
class BatchResult:
    scores: np.ndarray           # [n, max_labels] f32
    labels: np.ndarray           # [n] int32 (-1 for token_tag)
    tags: np.ndarray | None      # [n, stride] int32 (-1 beyond each request)
    trace: list = field(default_factory=list)  # LoadRecord dicts


class GpuEngine:
    """One CUDA context (one GPU) of the hPLM serving backend."""

    def __init__(self, cfg: ModelConfig, higher_f32: np.ndarray, *, device: int = 0,
                 precision: int = 0, max_batch: int = 256, max_seq: int = 128,
                 bottleneck: int = 64, max_labels: int = 8, pipeline_mode: int = MODE_FINE,
                 pool_bytes: int = 0, max_tasks: int = 1024, max_instances: int = 0,
                 max_heads: int = 0, max_versions: int = 64, max_new_tokens: int = 0):
        self.cfg = cfg
        self.max_labels = max_labels
        self._pending: dict[int, int] = {}
        self.max_batch = max_batch
        self.max_seq = max_seq
        self.bottleneck = bottleneck
        self.max_tasks = max_tasks
        self.max_instances = max_instances or max_tasks
        self.max_heads = max_heads or max_tasks
        self.max_versions = max_versions
        opts = Options(precision, max_batch, max_seq, bottleneck, max_labels, pipeline_mode,
                       pool_bytes, max_tasks, max_instances or max_tasks, max_heads or max_tasks,
                       max_versions, max_new_tokens, 0)
        hi = np.ascontiguousarray(higher_f32, np.float32)
        assert hi.size == cfg.higher_layers * layer_floats(cfg), "higher weights size"
        h = ctypes.c_void_p()
        check(_native.lib().hmi_gpu_create(device, ctypes.byref(cfg), ctypes.byref(opts),
                                           _p(hi, ctypes.c_float), ctypes.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            _native.lib().hmi_gpu_destroy(self.h)
            self.h = None

    __del__ = close

    # ---- registration ----------------------------------------------------
    def upload_table(self, version: int, parent: int, key_len, keys, reps) -> None:
        kl = np.ascontiguousarray(key_len, np.uint32)
        k = np.ascontiguousarray(keys, np.uint32)
        r = np.ascontiguousarray(reps, np.float32)
        check(_native.lib().hmi_gpu_upload_table(self.h, version, parent & 0xFFFFFFFF, len(kl),
                                                 _p(kl, ctypes.c_uint32), _p(k, ctypes.c_uint32),
                                                 _p(r, ctypes.c_float)))

    def register_task(self, task: int, adapter_f32) -> None:
        a = np.ascontiguousarray(adapter_f32, np.float32)
        check(_native.lib().hmi_gpu_register_task(self.h, task, _p(a, ctypes.c_float)))

    def register_tasks(self, tasks, adapters, threads: int = 0) -> None:
        """Bulk register_set on host threads (all-or-nothing)."""
        idx = np.ascontiguousarray(tasks, np.uint32)
        arrs = [np.ascontiguousarray(a, np.float32) for a in adapters]
        assert len(arrs) == len(idx)
        ptrs = (ctypes.POINTER(ctypes.c_float) * max(1, len(arrs)))(*[_p(a, ctypes.c_float) for a in arrs])
        check(_native.lib().hmi_gpu_register_tasks(self.h, len(idx), _p(idx, ctypes.c_uint32), ptrs,
                                                   threads))

    def register_task_files(self, tasks, paths, threads: int = 0) -> None:
        """Bulk register_set from ADP1 files read and converted on host threads."""
        idx = np.ascontiguousarray(tasks, np.uint32)
        enc = [p.encode() for p in paths]
        assert len(enc) == len(idx)
        arr = (ctypes.c_char_p * max(1, len(enc)))(*enc)
        check(_native.lib().hmi_gpu_register_task_files(self.h, len(idx), _p(idx, ctypes.c_uint32),
                                                        arr, threads))

    def replace_task(self, task: int, adapter_f32) -> None:
        a = np.ascontiguousarray(adapter_f32, np.float32)
        check(_native.lib().hmi_gpu_replace_task(self.h, task, _p(a, ctypes.c_float)))

    def unregister_task(self, task: int) -> None:
        check(_native.lib().hmi_gpu_unregister_task(self.h, task))

    # ---- peer rebalancing of tenants' adapters
    def export_task(self, task: int) -> bytes:
        """Pins every layer of ``task`` resident in this engine's HBM slot pool and returns the
        hmi_task_export record (bytes: it crosses processes as-is) until release_export."""
        ex = _native.TaskExport()
        check(_native.lib().hmi_gpu_export_task(self.h, task, ctypes.byref(ex)))
        return bytes(ex)

    def import_task(self, task: int, export: bytes, adapter_f32=None) -> int:
        """Registers ``task`` here with its HBM slots copied device to device from the exporting
        engine (same process: peer copy; another process: CUDA IPC). Returns the bytes moved."""
        ex = _native.TaskExport.from_buffer_copy(export)
        a = None if adapter_f32 is None else np.ascontiguousarray(adapter_f32, np.float32)
        moved = ctypes.c_uint64(0)
        check(_native.lib().hmi_gpu_import_task(self.h, task, ctypes.byref(ex),
                                                None if a is None else _p(a, ctypes.c_float),
                                                ctypes.byref(moved)))
        return int(moved.value)

    def release_export(self, task: int, drop: bool = False) -> None:
        check(_native.lib().hmi_gpu_release_export(self.h, task, int(drop)))

    def migrate_task(self, dst: "GpuEngine", task: int, keep_source: bool = False) -> int:
        """Moves (or, keep_source=True, replicates) a task's adapter set to ``dst`` over the
        device interconnect; the source keeps serving it until the import has landed."""
        ex = self.export_task(task)
        try:
            moved = dst.import_task(task, ex)
        except BaseException:
            self.release_export(task, drop=False)
            raise
        self.release_export(task, drop=not keep_source)
        return moved

    def register_head(self, head: int, kind: int, w, b) -> None:
        w = np.ascontiguousarray(w, np.float32)
        b = np.ascontiguousarray(b, np.float32)
        check(_native.lib().hmi_gpu_register_head(self.h, head, kind, b.shape[0],
                                                  _p(w, ctypes.c_float), _p(b, ctypes.c_float)))

    def bind_instance(self, instance: int, version: int, task: int, head: int) -> None:
        check(_native.lib().hmi_gpu_bind_instance(self.h, instance, version, task, head))

    def unbind_instance(self, instance: int) -> None:
        check(_native.lib().hmi_gpu_unbind_instance(self.h, instance))

    # ---- serving ---------------------------------------------------------
    def infer_batch(self, instance_idx, tokens, lens, *, want_tags: bool = False,
                    want_trace: bool = False) -> BatchResult:
        inst = np.ascontiguousarray(instance_idx, np.uint32)
        toks = np.ascontiguousarray(tokens, np.uint32)
        ln = np.ascontiguousarray(lens, np.uint32)
        n = inst.shape[0]
        stride = toks.shape[1]
        scores = np.zeros((n, self.max_labels), np.float32)
        labels = np.zeros(n, np.int32)
        tags = np.zeros((n, stride), np.int32) if want_tags else None
        cap = n * self.cfg.higher_layers * 2 + 16 if want_trace else 0
        recs = (LoadRecord * max(cap, 1))()
        ev = np.zeros(max(cap * self.cfg.higher_layers, 1), np.uint32)
        nt = ctypes.c_uint32(0)
        L = _native.lib()
        check(L.hmi_gpu_infer_batch(self.h, n, _p(inst, ctypes.c_uint32), _p(toks, ctypes.c_uint32),
                                    stride, _p(ln, ctypes.c_uint32), _p(scores, ctypes.c_float),
                                    _p(labels, ctypes.c_int32), _p(tags, ctypes.c_int32),
                                    recs if want_trace else None, cap,
                                    _p(ev, ctypes.c_uint32) if want_trace else None, ev.size,
                                    ctypes.byref(nt) if want_trace else None))
        trace = []
        if want_trace:
            for i in range(nt.value):
                r = recs[i]
                trace.append({"task": r.task, "layer": r.layer, "hit": bool(r.hit),
                              "bytes": r.bytes,
                              "evicted": [int(x) for x in ev[r.evicted_offset:r.evicted_offset + r.n_evicted]]})
        return BatchResult(scores, labels, tags, trace)

    def upload_plt1(self, path: str, streamed: bool = True) -> tuple[int, int]:
        """VersionTree::add_branch from a PLT1 file (plot_io.cpp:35-72); (version, parent).
        streamed: chunked pinned reads shipped to the GPU whole, rows scattered on the device
        (hmi_gpu_upload_plt1); else load the table on the host, then upload it."""
        L = _native.lib()
        v, p = ctypes.c_uint32(0), ctypes.c_uint32(0)
        if streamed:
            check(L.hmi_gpu_upload_plt1(self.h, path.encode(), ctypes.byref(v), ctypes.byref(p)))
            return v.value, p.value
        h = ctypes.c_void_p()
        check(L.hmi_plot_table_load(path.encode(), ctypes.byref(h), ctypes.byref(v), ctypes.byref(p),
                                    None))
        try:
            check(L.hmi_gpu_upload_plot_table(self.h, v.value, p.value, h))
        finally:
            L.hmi_plot_table_free(h)
        return v.value, p.value

    def register_task_file(self, task: int, path: str) -> None:
        """AdapterStore::register_set from an ADP1 file (adapter_set.cpp:48-75)."""
        check(_native.lib().hmi_gpu_register_task_file(self.h, task, path.encode()))

    STAGES = ("retrieve", "prefetch", "compute", "head", "host")
    WORKERS = ("cpu", "io", "compute")

    def trace(self, enable: bool) -> None:
        """Start (clearing) or stop StageTrace recording (hmi_gpu_trace)."""
        check(_native.lib().hmi_gpu_trace(self.h, int(enable)))

    def stage_trace(self) -> list:
        """StageTrace records: dicts {batch, stage, layer, worker, start_ms, end_ms}."""
        L = _native.lib()
        n = ctypes.c_uint32(0)
        check(L.hmi_gpu_stage_trace(self.h, None, 0, ctypes.byref(n)))
        recs = (_native.StageRecord * max(n.value, 1))()
        check(L.hmi_gpu_stage_trace(self.h, recs, n.value, ctypes.byref(n)))
        return [{"batch": int(r.batch), "stage": self.STAGES[r.stage], "layer": int(r.layer),
                 "worker": self.WORKERS[r.worker], "start_ms": r.start_ms, "end_ms": r.end_ms}
                for r in recs[:n.value]]

    def submit_batch(self, instance_idx, tokens, lens) -> int:
        """Enqueue a batch (host buffers) and return its ticket at once (hmi_gpu_submit_batch)."""
        inst = np.ascontiguousarray(instance_idx, np.uint32)
        toks = np.ascontiguousarray(tokens, np.uint32)
        ln = np.ascontiguousarray(lens, np.uint32)
        t = ctypes.c_uint64(0)
        check(_native.lib().hmi_gpu_submit_batch(self.h, inst.shape[0], _p(inst, ctypes.c_uint32),
                                                 _p(toks, ctypes.c_uint32), toks.shape[1],
                                                 _p(ln, ctypes.c_uint32), ctypes.byref(t)))
        self._pending[t.value] = inst.shape[0]
        return t.value

    def wait_batch(self, ticket: int) -> BatchResult:
        """Block until a submitted batch finished; its scores and labels (hmi_gpu_wait_batch)."""
        n = self._pending.pop(ticket)
        scores = np.zeros((n, self.max_labels), np.float32)
        labels = np.zeros(n, np.int32)
        check(_native.lib().hmi_gpu_wait_batch(self.h, ticket, _p(scores, ctypes.c_float),
                                               _p(labels, ctypes.c_int32)))
        return BatchResult(scores, labels, None, [])

    def infer_batch_device(self, instance_idx, d_tokens: int, stride: int, d_lens: int,
                           max_len: int, d_scores: int, d_labels: int) -> None:
        inst = np.ascontiguousarray(instance_idx, np.uint32)
        check(_native.lib().hmi_gpu_infer_batch_device(
            self.h, inst.shape[0], _p(inst, ctypes.c_uint32), ctypes.c_void_p(d_tokens), stride,
            ctypes.c_void_p(d_lens), max_len, ctypes.c_void_p(d_scores), ctypes.c_void_p(d_labels)))

    def generate(self, instance_idx, tokens, lens, n_new: int):
        """Greedy continuation of causal prompts through a wide lm head
        (hmi_gpu_generate): returns (tokens [n, n_new] int32, logits [n, n_new] f32)."""
        inst = np.ascontiguousarray(instance_idx, np.uint32)
        toks = np.ascontiguousarray(tokens, np.uint32)
        ln = np.ascontiguousarray(lens, np.uint32)
        n = inst.shape[0]
        out = np.zeros((n, n_new), np.int32)
        logit = np.zeros((n, n_new), np.float32)
        check(_native.lib().hmi_gpu_generate(self.h, n, _p(inst, ctypes.c_uint32),
                                             _p(toks, ctypes.c_uint32), toks.shape[1],
                                             _p(ln, ctypes.c_uint32), n_new,
                                             _p(out, ctypes.c_int32), _p(logit, ctypes.c_float)))
        return out, logit

    def synchronize(self) -> None:
        check(_native.lib().hmi_gpu_synchronize(self.h))

    @property
    def stream(self) -> int:
        return int(_native.lib().hmi_gpu_stream(self.h) or 0)

    # ---- introspection ---------------------------------------------------
    def debug_routing(self, n: int):
        L = self.cfg.higher_layers
        v = np.zeros(n, np.int32)
        t = np.zeros(n, np.int32)
        hd = np.zeros(n, np.int32)
        s = np.zeros((L, n), np.int32)
        check(_native.lib().hmi_gpu_debug_routing(self.h, _p(v, ctypes.c_int32), _p(t, ctypes.c_int32),
                                                  _p(hd, ctypes.c_int32), _p(s, ctypes.c_int32)))
        return v, t, hd, s

    def debug_gather(self, n: int):
        S = ctypes.c_uint32(0)
        check(_native.lib().hmi_gpu_debug_gather(self.h, None, None, ctypes.byref(S)))
        ng = self.cfg.max_fragment
        rows = np.zeros((n, S.value, ng), np.int32)
        lev = np.zeros((n, S.value, ng), np.int32)
        check(_native.lib().hmi_gpu_debug_gather(self.h, _p(rows, ctypes.c_int32),
                                                 _p(lev, ctypes.c_int32), ctypes.byref(S)))
        return rows, lev

    def set_debug(self, flags: int) -> None:
        check(_native.lib().hmi_gpu_set_debug(self.h, flags))

    def debug_h0(self, n: int, S: int) -> np.ndarray:
        out = np.zeros((n, S, self.cfg.hidden_size), np.float64)
        check(_native.lib().hmi_gpu_debug_h0(self.h, _p(out, ctypes.c_double)))
        return out

    def debug_hidden(self, n: int, S: int) -> np.ndarray:
        out = np.zeros((n, S, self.cfg.hidden_size), np.float32)
        check(_native.lib().hmi_gpu_debug_hidden(self.h, _p(out, ctypes.c_float)))
        return out

    def pool_stats(self) -> dict:
        o = np.zeros(8, np.uint64)
        check(_native.lib().hmi_gpu_pool_stats(self.h, _p(o, ctypes.c_uint64)))
        keys = ("hits", "loads", "resident_bytes", "max_resident_bytes_seen",
                "resident_task_count", "capacity_bytes", "physical_slots", "bytes_copied")
        return {k: int(v) for k, v in zip(keys, o)}

    def pool_slot(self, task: int, layer: int) -> int:
        s = ctypes.c_int32(0)
        check(_native.lib().hmi_gpu_pool_slot(self.h, task, layer, ctypes.byref(s)))
        return s.value

    def profile(self, enable: bool) -> None:
        check(_native.lib().hmi_gpu_profile(self.h, int(enable)))

    def profile_read(self) -> dict:
        n = 16
        ms = np.zeros(n, np.float64)
        cnt = np.zeros(n, np.uint64)
        L = _native.lib()
        check(L.hmi_gpu_profile_read(self.h, _p(ms, ctypes.c_double), _p(cnt, ctypes.c_uint64)))
        return {L.hmi_gpu_profile_name(i).decode(): (float(ms[i]), int(cnt[i])) for i in range(n)}


class SlotPoolPolicy:
    """Standalone DeviceSlotPool policy (host only) for trace-parity tests."""

    def __init__(self, capacity_bytes: int, physical_slots: int = 0, block_len: int = 1):
        h = ctypes.c_void_p()
        if physical_slots:  # with the engine's physical slot placement
            check(_native.lib().hmi_pool_create_placed(capacity_bytes, physical_slots, block_len,
                                                       ctypes.byref(h)))
        else:
            check(_native.lib().hmi_pool_create(capacity_bytes, ctypes.byref(h)))
        self.h = h

    def slot(self, task: int, layer: int) -> int:
        s = ctypes.c_int32(-1)
        check(_native.lib().hmi_pool_slot(self.h, task, layer, ctypes.byref(s)))
        return s.value

    def __del__(self):
        if getattr(self, "h", None):
            _native.lib().hmi_pool_destroy(self.h)
            self.h = None

    def register(self, task: int, layers: int, layer_bytes: int) -> None:
        check(_native.lib().hmi_pool_register(self.h, task, layers, layer_bytes))

    def op(self, op: int, tasks, layer: int = 0):
        t = np.ascontiguousarray(tasks, np.uint32)
        cap = max(len(t), 1)
        recs = (LoadRecord * cap)()
        ev = np.zeros(4096, np.uint32)
        n = ctypes.c_int32(0)
        check(_native.lib().hmi_pool_op(self.h, op, len(t), _p(t, ctypes.c_uint32), layer, recs,
                                        cap, _p(ev, ctypes.c_uint32), ev.size, ctypes.byref(n)))
        if n.value < 0:
            return None
        if op >= 2:
            return n.value
        out = []
        for i in range(n.value):
            r = recs[i]
            out.append({"task": r.task, "hit": bool(r.hit), "bytes": int(r.bytes),
                        "evicted": [int(x) for x in ev[r.evicted_offset:r.evicted_offset + r.n_evicted]]})
        return out

    def ensure_resident(self, tasks):
        return self.op(0, tasks)

    def try_ensure_layer_resident(self, tasks, layer):
        return self.op(1, tasks, layer)

    def pin(self, tasks):
        self.op(2, tasks)

    def unpin(self, tasks):
        self.op(3, tasks)

    def touch(self, tasks):
        self.op(4, tasks)

    def evict(self, task) -> bool:
        return bool(self.op(5, [task]))

    def stats(self) -> dict:
        o = np.zeros(8, np.uint64)
        check(_native.lib().hmi_pool_stats(self.h, _p(o, ctypes.c_uint64)))
        keys = ("hits", "loads", "resident_bytes", "max_resident_bytes_seen",
                "resident_task_count", "capacity_bytes")
        return {k: int(v) for k, v in zip(keys, o)}


# ---------------------------------------------------------------------------
# seeded generators (weights.cpp:72-118, adapter_set.cpp:15-25)
# ---------------------------------------------------------------------------
def generate_higher(cfg: ModelConfig) -> np.ndarray:
    """Higher-stack weights of generate_model(cfg), f32, HMI1 per-layer order."""
    out = np.empty((cfg.higher_layers, layer_floats(cfg)), np.float32)
    check(_native.lib().hmi_generate_model(ctypes.byref(cfg), None, None, None,
                                           _p(out, ctypes.c_float)))
    return out


def generate_adapter(cfg: ModelConfig, r: int, seed: int) -> np.ndarray:
    out = np.empty((cfg.higher_layers, adapter_layer_floats(cfg, r)), np.float32)
    check(_native.lib().hmi_generate_adapter(ctypes.byref(cfg), r, seed, _p(out, ctypes.c_float)))
    return out


def generate_head(d: int, labels: int, seed: int):
    w = np.empty((d, labels), np.float32)
    b = np.empty((labels,), np.float32)
    check(_native.lib().hmi_generate_head(d, labels, seed, _p(w, ctypes.c_float),
                                          _p(b, ctypes.c_float)))
    return w, b


def engine_counters(eng: GpuEngine) -> dict:
    o = np.zeros(4, np.uint64)
    check(_native.lib().hmi_gpu_counters(eng.h, _p(o, ctypes.c_uint64)))
    return {"launches": int(o[0]), "batches": int(o[1]), "adapter_copies": int(o[2]),
            "numa_node": None if int(o[3]) == 2**64 - 1 else int(o[3])}


def h2d_probe(eng: GpuEngine, nbytes: int = 256 << 20, reps: int = 8) -> float:
    """GB/s of pinned (NUMA-local) host -> HBM copies on the engine's copy stream."""
    g = ctypes.c_double(0.0)
    check(_native.lib().hmi_gpu_h2d_probe(eng.h, ctypes.c_uint64(nbytes), reps, ctypes.byref(g)))
    return g.value
