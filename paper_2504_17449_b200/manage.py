# SPDX-License-Identifier: Apache-2.0
"""The ``manage`` half of the service (SPEC.md service module,
S:503-579): domain and instance lifecycle over one GPU engine, with between-batch atomicity.

* ``create_domain``   derive_branch on the GPU builder from a tenant corpus (minimum corpus size,
                      S:527 "only domain data with a certain size of corpus"; default 10,000
                      tokens) and registration of the branch in the version tree
* ``update_domain``   re-derivation from the merged corpus: a new table version under the same
                      domain label; the tenant's instances move to it
* ``create_instance`` adapter registration (array, ADP1 file or seeded generation), output head,
                      binding to a version
* ``update_instance`` adapter replacement ("replaces the adapter set atomically between
                      batches")
* ``delete_instance`` registry removal, adapter host entry dropped, device slot evicted
* ``snapshot_state``  JSON view of the registry and version tree; ``save`` / ``load`` round-trip
                      it through PLT1 / ADP1 artefacts

Mutations are queued by ``submit`` (any thread) and applied by ``apply_pending``, which
``serving.Server`` calls before each batch, so no batch ever sees half an operation
(S:565 concurrency model). The HTTP wire format of S:553 is out of scope (SURVEY.md §8:
networking). Errors: unknown ids -> RoutingError (404 class), duplicate create -> ConflictError,
corpus below threshold or malformed payload -> ValidationError.
"""
from __future__ import annotations

import json
import os
import threading
from collections import deque
from dataclasses import dataclass, field

import numpy as np

from . import plot
from ._native import ConflictError, RoutingError
from .engine import generate_adapter, generate_head
from .serving import InstanceBinding, Registry

OPS = ("create_domain", "update_domain", "create_instance", "update_instance", "delete_instance")
ROOT_PARENT = 0xFFFFFFFF


class ValidationError(ValueError):
    pass


@dataclass
class ManageRequest:
    op: str
    tenant_id: str
    payload: dict = field(default_factory=dict)


@dataclass
class ManageResult:
    status: str = "ok"
    version_id: int | None = None
    instance_id: str | None = None


class ManageTicket:
    def __init__(self, req: ManageRequest):
        self.req = req
        self._done = threading.Event()
        self._result: ManageResult | None = None
        self._error: BaseException | None = None

    def done(self) -> bool:
        return self._done.is_set()

    def result(self, timeout: float | None = None) -> ManageResult:
        if not self._done.wait(timeout):
            raise TimeoutError("manage request not applied yet (no batch boundary reached)")
        if self._error is not None:
            raise self._error
        return self._result


@dataclass
class _Version:
    parent: int | None
    label: str
    tenant: str | None
    table: dict
    corpus: list | None = None
    alpha: float = 0.0


@dataclass
class _Instance:
    tenant: str
    version: int
    task: int
    head: int
    adapter_ref: dict  # {"array": ...} | {"file": path} | {"seed": int}
    head_ref: dict


class Manager:
    def __init__(self, engine, builder, root_table: dict, registry: Registry | None = None, *,
                 alpha: float = 50.0, min_corpus_tokens: int = 10_000):
        self.engine, self.builder = engine, builder
        self.registry = registry if registry is not None else Registry()
        self.alpha, self.min_corpus_tokens = float(alpha), int(min_corpus_tokens)
        self.versions: dict[int, _Version] = {}
        self.tenants: dict[str, set] = {}
        self.instances: dict[str, _Instance] = {}
        self._free_inst = list(range(engine.max_instances - 1, -1, -1))
        self._free_task = list(range(engine.max_tasks - 1, -1, -1))
        self._next_head = 0  # heads are immutable on the device: indices are not reused
        self._pending: deque[ManageTicket] = deque()
        self._mu = threading.Lock()
        self._state_mu = threading.Lock()
        engine.upload_table(0, ROOT_PARENT, root_table["key_len"], root_table["keys"],
                            root_table["reps"])
        self.versions[0] = _Version(None, "root", None, root_table)

    # ---- request plumbing
    def submit(self, req: ManageRequest) -> ManageTicket:
        if req.op not in OPS:
            raise ValidationError(f"unknown manage op {req.op!r}")
        t = ManageTicket(req)
        with self._mu:
            self._pending.append(t)
        return t

    def apply_pending(self) -> int:
        """Applies every queued request in submission order (a batch boundary)."""
        with self._mu:
            todo = list(self._pending)
            self._pending.clear()
        for t in todo:
            try:
                with self._state_mu:
                    t._result = getattr(self, "_" + t.req.op)(t.req.tenant_id, t.req.payload)
            except BaseException as e:  # noqa: BLE001 - delivered to the caller through the ticket
                t._error = e
            t._done.set()
        return len(todo)

    def handle(self, req: ManageRequest) -> ManageResult:
        """Submit and apply now (callers outside a serving loop)."""
        t = self.submit(req)
        self.apply_pending()
        return t.result()

    # ---- ops
    def _corpus(self, payload, have: int = 0) -> list:
        corpus = payload.get("corpus")
        if corpus is None:
            raise ValidationError("payload needs 'corpus'")
        corpus = [np.asarray(s, np.uint32) for s in corpus]
        n = sum(len(s) for s in corpus) + have
        if n < self.min_corpus_tokens:
            raise ValidationError(f"domain corpus of {n} tokens is below the minimum of "
                                  f"{self.min_corpus_tokens}")
        return corpus

    def _new_version_id(self) -> int:
        vid = max(self.versions) + 1
        if vid >= self.engine.max_versions:
            raise ValidationError("version tree is full (max_versions)")
        return vid

    def _create_domain(self, tenant, payload) -> ManageResult:
        label = payload.get("label", tenant)
        if any(v.tenant == tenant and v.label == label for v in self.versions.values()):
            raise ConflictError(f"domain {label!r} of tenant {tenant!r} already exists")
        base = int(payload.get("base_version", 0))
        if base not in self.versions:
            raise RoutingError(f"version {base} does not exist")
        corpus = self._corpus(payload)
        alpha = float(payload.get("alpha", self.alpha))
        return ManageResult(version_id=self._derive(tenant, label, base, corpus, alpha))

    def _derive(self, tenant, label, base, corpus, alpha) -> int:
        vid = self._new_version_id()
        table = self.builder.derive_branch(self.versions[base].table, corpus, alpha)
        self.engine.upload_table(vid, base, table["key_len"], table["keys"], table["reps"])
        self.versions[vid] = _Version(base, label, tenant, table, corpus, alpha)
        return vid

    def _update_domain(self, tenant, payload) -> ManageResult:
        old = int(payload.get("version_id", -1))
        v = self.versions.get(old)
        if v is None or v.tenant != tenant:
            raise RoutingError(f"version {old} is not a domain of tenant {tenant!r}")
        corpus = v.corpus + self._corpus(payload, have=sum(len(x) for x in v.corpus))
        vid = self._derive(tenant, v.label, v.parent, corpus, v.alpha)
        v.label = f"{v.label}@{old}"  # superseded; the label now names the new version
        for iid in sorted(self.tenants.get(tenant, ())):
            inst = self.instances[iid]
            if inst.version == old:
                idx = self.registry.instances[iid]
                self.engine.unbind_instance(idx)
                self.engine.bind_instance(idx, vid, inst.task, inst.head)
                inst.version = vid
                self.registry.bindings[iid].version_id = vid
        return ManageResult(version_id=vid)

    def _adapter(self, payload):
        if "adapter" in payload:
            return np.ascontiguousarray(payload["adapter"], np.float32), {"array": True}
        if "adapter_file" in payload:
            return None, {"file": str(payload["adapter_file"])}
        if "adapter_seed" in payload:
            seed = int(payload["adapter_seed"])
            return generate_adapter(self.engine.cfg, self.engine.bottleneck, seed), {"seed": seed}
        raise ValidationError("payload needs 'adapter', 'adapter_file' or 'adapter_seed'")

    def _create_instance(self, tenant, payload) -> ManageResult:
        iid = payload.get("instance_id")
        if not iid:
            raise ValidationError("payload needs 'instance_id'")
        if iid in self.instances:
            raise ConflictError(f"instance {iid!r} already exists")
        vid = int(payload.get("version_id", 0))
        if vid not in self.versions or self.versions[vid].tenant not in (None, tenant):
            raise RoutingError(f"version {vid} is not available to tenant {tenant!r}")
        body, aref = self._adapter(payload)
        if "head" in payload:
            h = payload["head"]
            kind, w, b = int(h.get("kind", 0)), h["w"], h["b"]
            href = {"kind": kind, "w": np.asarray(w, np.float32), "b": np.asarray(b, np.float32)}
        else:
            kind = int(payload.get("head_kind", 0))
            labels, seed = int(payload.get("labels", self.engine.max_labels)), int(payload.get("head_seed", 0))
            w, b = generate_head(self.engine.cfg.hidden_size, labels, seed)
            href = {"kind": kind, "labels": labels, "seed": seed}
        want = payload.get("_indices")  # (task, instance, head) of a saved snapshot (load())
        if want is not None:
            task, inst_idx, head = (int(x) for x in want)
            if task not in self._free_task or inst_idx not in self._free_inst or not 0 <= head < self.engine.max_heads:
                raise ConflictError(f"indices {want} of instance {iid!r} are not free")
            self._free_task.remove(task)
            self._free_inst.remove(inst_idx)
        else:
            if not self._free_inst or not self._free_task or self._next_head >= self.engine.max_heads:
                raise ValidationError("engine capacity reached (max_instances / max_tasks / max_heads)")
            task, inst_idx, head = self._free_task.pop(), self._free_inst.pop(), self._next_head
        try:
            if body is None:
                self.engine.register_task_file(task, aref["file"])
            else:
                self.engine.register_task(task, body)
            try:
                self.engine.register_head(head, kind, w, b)
                self._next_head = max(self._next_head, head + 1)
                self.engine.bind_instance(inst_idx, vid, task, head)
            except BaseException:
                self.engine.unregister_task(task)
                raise
        except BaseException:
            self._free_task.append(task)
            self._free_inst.append(inst_idx)
            raise
        if aref.get("array"):
            aref = {"array": body}
        self.instances[iid] = _Instance(tenant, vid, task, head, aref, href)
        self.tenants.setdefault(tenant, set()).add(iid)
        self.registry.tasks[iid] = task
        self.registry.heads[iid] = head
        self.registry.instances[iid] = inst_idx
        self.registry.bindings[iid] = InstanceBinding(vid, iid, iid)
        return ManageResult(instance_id=iid)

    def _owned(self, tenant, payload) -> _Instance:
        iid = payload.get("instance_id")
        inst = self.instances.get(iid)
        if inst is None or inst.tenant != tenant:
            raise RoutingError(f"instance {iid!r} of tenant {tenant!r} does not exist")
        return inst

    def _update_instance(self, tenant, payload) -> ManageResult:
        inst = self._owned(tenant, payload)
        body, aref = self._adapter(payload)
        if body is None:
            body = plot.load_adp1(aref["file"])[1]
        self.engine.replace_task(inst.task, body)
        inst.adapter_ref = {"array": body} if aref.get("array") else aref
        return ManageResult(instance_id=payload["instance_id"])

    def _delete_instance(self, tenant, payload) -> ManageResult:
        inst = self._owned(tenant, payload)
        iid = payload["instance_id"]
        idx = self.registry.instances.pop(iid)
        self.engine.unbind_instance(idx)
        self.engine.unregister_task(inst.task)
        self._free_inst.append(idx)
        self._free_task.append(inst.task)
        del self.registry.bindings[iid], self.registry.tasks[iid], self.registry.heads[iid]
        del self.instances[iid]
        self.tenants[tenant].discard(iid)
        return ManageResult(instance_id=iid)

    # ---- state
    def snapshot_state(self) -> dict:
        with self._state_mu:
            return {
                "versions": {str(k): {"parent": v.parent, "label": v.label, "tenant": v.tenant,
                                      "entries": int(len(v.table["key_len"])), "alpha": v.alpha}
                             for k, v in sorted(self.versions.items())},
                "tenants": {t: sorted(s) for t, s in sorted(self.tenants.items())},
                "instances": {i: {"tenant": x.tenant, "version": x.version, "task": x.task,
                                  "head": x.head, "index": self.registry.instances[i]}
                              for i, x in sorted(self.instances.items())},
            }

    def save(self, directory: str) -> None:
        """Snapshot plus the artefacts to rebuild it: PLT1 per version, the domain corpora,
        ADP1 per array-registered adapter, head weights."""
        os.makedirs(directory, exist_ok=True)
        snap = self.snapshot_state()
        cfg = self.engine.cfg
        for k, v in self.versions.items():
            plot.save_plt1(v.table, os.path.join(directory, f"v{k}.plt1"), k,
                           ROOT_PARENT if v.parent is None else v.parent, v.label,
                           int(round(v.alpha * 100)))
            if v.corpus is not None:
                np.savez(os.path.join(directory, f"v{k}.corpus.npz"), *v.corpus)
        refs = {}
        for iid, x in self.instances.items():
            stem = f"i{x.task}"
            a = x.adapter_ref
            if "array" in a:
                plot.save_adp1(os.path.join(directory, stem + ".adp1"), iid, a["array"],
                               cfg.hidden_size, self.engine.bottleneck)
                a = {"file": stem + ".adp1", "relative": True}
            h = dict(x.head_ref)
            if "w" in h:
                np.savez(os.path.join(directory, stem + ".head.npz"), w=h.pop("w"), b=h.pop("b"))
                h["file"] = stem + ".head.npz"
            refs[iid] = {"adapter": a, "head": h}
        snap["artefacts"] = refs
        with open(os.path.join(directory, "state.json"), "w") as f:
            json.dump(snap, f, indent=1, sort_keys=True)

    @classmethod
    def load(cls, directory: str, engine, builder, registry: Registry | None = None, **kw) -> "Manager":
        with open(os.path.join(directory, "state.json")) as f:
            snap = json.load(f)
        root, _, _, _ = plot.load_plt1(os.path.join(directory, "v0.plt1"))
        m = cls(engine, builder, root, registry, **kw)
        for k in sorted(int(x) for x in snap["versions"] if x != "0"):
            v = snap["versions"][str(k)]
            table, vid, parent, _ = plot.load_plt1(os.path.join(directory, f"v{k}.plt1"))
            engine.upload_table(vid, parent, table["key_len"], table["keys"], table["reps"])
            cp = os.path.join(directory, f"v{k}.corpus.npz")
            corpus = None
            if os.path.exists(cp):
                z = np.load(cp)
                corpus = [z[f"arr_{i}"] for i in range(len(z.files))]
            m.versions[vid] = _Version(v["parent"], v["label"], v["tenant"], table, corpus, v["alpha"])
        for iid, x in sorted(snap["instances"].items(), key=lambda kv: kv[1]["task"]):
            ref = snap["artefacts"][iid]
            p = {"instance_id": iid, "version_id": x["version"],
                 "_indices": (x["task"], x["index"], x["head"])}
            a = ref["adapter"]
            if "file" in a:
                p["adapter_file"] = os.path.join(directory, a["file"]) if a.get("relative") else a["file"]
            else:
                p["adapter_seed"] = a["seed"]
            h = ref["head"]
            if "file" in h:
                z = np.load(os.path.join(directory, h["file"]))
                p["head"] = {"kind": h["kind"], "w": z["w"], "b": z["b"]}
            else:
                p.update(head_kind=h["kind"], labels=h["labels"], head_seed=h["seed"])
            m.handle(ManageRequest("create_instance", x["tenant"], p))
        return m
