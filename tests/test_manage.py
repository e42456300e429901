# SPDX-License-Identifier: Apache-2.0
"""Manage front end (SPEC.md service module S:503-579).

CPU: the lifecycle and its errors, between-batch atomicity and queue conservation in the Server,
and the save / load round trip, over a recording stand-in engine (tables from the product's own
key selection). GPU: the SPEC's examples end to end on the B200 engine and PLOT builder —
create_domain at alpha 50 then infer through the branch matches the oracle, 9 requests at
max_batch 3 give 3 batches, two instances differing only in adapters differ, a tenant's manage
ops never change another tenant's outputs (bit for bit), save / load reproduces routing, and
10,000 instances under one backbone register with pool residency inside its capacity."""
import numpy as np
import pytest

import oracle
from paper_2504_17449_b200 import engine as E
from paper_2504_17449_b200 import plot
from paper_2504_17449_b200._native import ConflictError, RoutingError
from paper_2504_17449_b200.engine import BatchResult
from paper_2504_17449_b200.manage import Manager, ManageRequest, ValidationError
from paper_2504_17449_b200.serving import InferRequest, Server

CFG = oracle.Config(128, 2, 2, 2, 256, 300, 0, 3, 5)
R, LABELS = 8, 5


def _corpus(seed, n_seq, length, lo=0, hi=300):
    rng = np.random.default_rng(seed)
    return [rng.integers(lo, hi, length).astype(np.uint32) for _ in range(n_seq)]


class FakeEngine:
    """Records the device state the manager drives; infer_batch returns, per request, a digest of
    (version, adapter, head) so tests can see which state a batch was served with."""

    def __init__(self, max_tasks=16, max_versions=8):
        self.cfg = E.model_config(*oracle.astuple(CFG))
        self.bottleneck, self.max_labels = R, LABELS
        self.max_tasks = self.max_instances = self.max_heads = max_tasks
        self.max_versions = max_versions
        self.tables, self.tasks, self.heads, self.binds = {}, {}, {}, {}
        self.calls = []

    def upload_table(self, v, parent, key_len, keys, reps):
        self.tables[v] = (parent, len(key_len))

    def register_task(self, t, a):
        if t in self.tasks:
            raise ConflictError("dup")
        self.tasks[t] = float(np.asarray(a, np.float64).sum())

    def register_task_file(self, t, path):
        self.register_task(t, plot.load_adp1(path)[1])

    def replace_task(self, t, a):
        if t not in self.tasks:
            raise RoutingError("no task")
        self.tasks[t] = float(np.asarray(a, np.float64).sum())

    def unregister_task(self, t):
        self.tasks.pop(t, None)

    def register_head(self, h, kind, w, b):
        if h in self.heads:
            raise ConflictError("dup head")
        self.heads[h] = float(np.asarray(w, np.float64).sum())

    def bind_instance(self, i, v, t, h):
        if v not in self.tables or t not in self.tasks or h not in self.heads:
            raise RoutingError("dangling")
        self.binds[i] = (v, t, h)

    def unbind_instance(self, i):
        self.binds.pop(i, None)

    def infer_batch(self, inst, toks, lens, want_tags=False):
        self.calls.append(len(inst))
        s = np.zeros((len(inst), LABELS), np.float32)
        for k, i in enumerate(inst):
            v, t, h = self.binds[int(i)]
            s[k, :3] = (v, self.tasks[t], self.heads[h])
        return BatchResult(s, np.zeros(len(inst), np.int32), None)


class FakeBuilder:
    def derive_branch(self, base, corpus, alpha):
        t = plot.select_branch(corpus, CFG.max_fragment, alpha)
        t["reps"] = np.zeros((int(t["key_len"].sum()), CFG.hidden_size), np.float32)
        return t


def _root():
    t = plot.select_root(_corpus(1, 4, 30), CFG.max_fragment, CFG.vocab_size)
    t["reps"] = np.zeros((int(t["key_len"].sum()), CFG.hidden_size), np.float32)
    return t


def _fake_manager(**kw):
    return Manager(FakeEngine(**kw), FakeBuilder(), _root(), min_corpus_tokens=200)


def _inst(m, tenant, iid, version, seed):
    return m.handle(ManageRequest("create_instance", tenant, {
        "instance_id": iid, "version_id": version, "adapter_seed": seed, "head_seed": seed + 100,
        "labels": LABELS})).instance_id


def test_lifecycle_and_errors():
    m = _fake_manager()
    snap = m.snapshot_state()
    assert list(snap["versions"]) == ["0"] and snap["tenants"] == {} and snap["instances"] == {}
    with pytest.raises(ValidationError):  # corpus below the minimum size
        m.handle(ManageRequest("create_domain", "A", {"corpus": _corpus(2, 2, 50)}))
    with pytest.raises(RoutingError):
        m.handle(ManageRequest("create_domain", "A", {"corpus": _corpus(2, 8, 50), "base_version": 7}))
    v1 = m.handle(ManageRequest("create_domain", "A", {"corpus": _corpus(2, 8, 50), "label": "law"})).version_id
    assert v1 == 1 and m.engine.tables[1][0] == 0
    with pytest.raises(ConflictError):
        m.handle(ManageRequest("create_domain", "A", {"corpus": _corpus(3, 8, 50), "label": "law"}))
    with pytest.raises(ValidationError):
        m.submit(ManageRequest("drop_everything", "A"))
    _inst(m, "A", "a1", v1, 1)
    with pytest.raises(ConflictError):
        _inst(m, "A", "a1", v1, 2)
    with pytest.raises(RoutingError):  # another tenant's domain
        _inst(m, "B", "b1", v1, 3)
    with pytest.raises(RoutingError):
        _inst(m, "B", "b1", 5, 3)
    _inst(m, "B", "b1", 0, 3)
    with pytest.raises(RoutingError):  # B cannot touch A's instance
        m.handle(ManageRequest("delete_instance", "B", {"instance_id": "a1"}))
    snap = m.snapshot_state()
    assert snap["tenants"] == {"A": ["a1"], "B": ["b1"]}
    assert snap["instances"]["a1"]["version"] == 1 and snap["versions"]["1"]["label"] == "law"
    # update_domain: new version under the same label; the tenant's instances move to it
    v2 = m.handle(ManageRequest("update_domain", "A", {"version_id": v1, "corpus": _corpus(4, 1, 10)})).version_id
    assert v2 == 2 and m.engine.binds[m.registry.instances["a1"]][0] == 2
    assert m.snapshot_state()["versions"]["2"]["label"] == "law"
    m.handle(ManageRequest("delete_instance", "A", {"instance_id": "a1"}))
    srv = Server(m.engine, m.registry, 3, 128, manager=m)
    with pytest.raises(RoutingError):
        srv.enqueue(InferRequest("r0", "A", "a1", [1, 2, 3]))
    assert len(m.engine.tasks) == 1 and len(m.engine.binds) == 1
    # indices are recycled: a new instance reuses the freed task / instance slots
    _inst(m, "A", "a2", v2, 5)
    assert m.snapshot_state()["instances"]["a2"]["task"] == snap["instances"]["a1"]["task"]


def test_between_batch_atomicity_and_conservation():
    m = _fake_manager()
    _inst(m, "A", "x", 0, 1)
    _inst(m, "B", "y", 0, 2)
    eng = m.engine
    srv = Server(eng, m.registry, 3, 128, manager=m)
    tickets = []
    orig = eng.infer_batch

    def hooked(inst, toks, lens, want_tags=False):
        out = orig(inst, toks, lens, want_tags)
        if len(eng.calls) == 1:  # a handler thread's requests arrive while batch 0 runs
            tickets.append(m.submit(ManageRequest("update_instance", "A",
                                                  {"instance_id": "x", "adapter_seed": 77})))
            tickets.append(m.submit(ManageRequest("delete_instance", "B", {"instance_id": "y"})))
        return out

    eng.infer_batch = hooked
    ids = ["x", "y", "x", "y", "x", "y", "x", "y", "x"]
    for k, iid in enumerate(ids):
        srv.enqueue(InferRequest(f"r{k}", "A" if iid == "x" else "B", iid, [1, 2, 3]))
    assert not tickets
    res = srv.run()
    assert all(t.done() for t in tickets)
    # batch 0 saw the old adapter; every later batch the new one; no batch mixed them
    old = [r.output.scores[1] for r in res if r.batch_id == 0 and r.request_id in ("r0", "r2")]
    new = [r.output.scores[1] for r in res if r.batch_id > 0]
    assert len(set(old)) == 1 and len(set(new)) == 1 and old[0] != new[0]
    # y was deleted at the boundary: its later requests are rejected, none lost or duplicated
    assert eng.calls == [3, 1, 2]  # batches (x y x) (y x y) (x y x), y gone after batch 0
    assert len(res) + len(srv.rejected) == len(ids)
    assert {r for r, _ in srv.rejected} == {"r3", "r5", "r7"}


def test_save_load_round_trip(tmp_path):
    m = _fake_manager()
    v = m.handle(ManageRequest("create_domain", "A", {"corpus": _corpus(2, 8, 50)})).version_id
    _inst(m, "A", "a", v, 1)
    m.handle(ManageRequest("create_instance", "B", {
        "instance_id": "b", "version_id": 0,
        "adapter": E.generate_adapter(m.engine.cfg, R, 9),
        "head": {"kind": 0, "w": np.ones((CFG.hidden_size, LABELS), np.float32), "b": np.zeros(LABELS, np.float32)}}))
    _inst(m, "A", "gone", v, 4)  # a deletion leaves holes the reload must reproduce
    m.handle(ManageRequest("delete_instance", "A", {"instance_id": "gone"}))
    _inst(m, "B", "c", 0, 5)
    m.save(str(tmp_path))
    m2 = Manager.load(str(tmp_path), FakeEngine(), FakeBuilder(), min_corpus_tokens=200)
    assert m2.snapshot_state() == m.snapshot_state()
    live = {x["head"] for x in m.snapshot_state()["instances"].values()}
    assert m2.engine.tasks == m.engine.tasks  # deleted instances' heads stay on the device
    assert m2.engine.heads == {h: w for h, w in m.engine.heads.items() if h in live}
    assert m2.engine.binds == m.engine.binds and m2.engine.tables == m.engine.tables
    # the reloaded domain keeps its corpus: update_domain still merges
    assert m2.handle(ManageRequest("update_domain", "A", {"version_id": v, "corpus": _corpus(5, 1, 9)})).version_id == 2


# ---------------------------------------------------------------------------------------- GPU
def _gpu_world(max_tasks=16, pool_bytes=0):
    mc = E.model_config(*oracle.astuple(CFG))
    eng = E.GpuEngine(mc, E.generate_higher(mc), max_batch=32, max_seq=128, bottleneck=R,
                      max_labels=LABELS, max_tasks=max_tasks, max_versions=8, pool_bytes=pool_bytes)
    b = plot.GpuPlotBuilder(mc)
    root = b.build_root(_corpus(1, 6, 40))
    return eng, b, Manager(eng, b, root, min_corpus_tokens=200)


def _requests(seed, n, hot):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n):
        k = int(rng.integers(3, 30))
        toks = rng.integers(0, CFG.vocab_size, k)
        s = int(rng.integers(0, max(1, k - 3)))
        toks[s:s + 3] = hot[int(rng.integers(0, len(hot)))]  # a fragment the branch holds
        out.append(toks.astype(np.uint32))
    return out


def _serve(srv, tenant, iids, reqs, tag):
    for k, (iid, t) in enumerate(zip(iids, reqs)):
        srv.enqueue(InferRequest(f"{tag}{k}", tenant[iid], iid, list(map(int, t))))
    return srv.run()


@pytest.mark.gpu
def test_gpu_manage_end_to_end(tmp_path):
    eng, b, m = _gpu_world()
    dom = _corpus(7, 10, 40, 20, 60)  # a narrow domain vocabulary: a concentrated branch
    v = m.handle(ManageRequest("create_domain", "A", {"corpus": dom, "alpha": 50.0})).version_id
    branch = m.versions[v].table
    assert len(branch["key_len"]) > 0
    _inst(m, "A", "x", v, 11)
    _inst(m, "B", "y", 0, 12)
    m.handle(ManageRequest("create_instance", "B", {"instance_id": "y2", "version_id": 0,
                                                    "adapter_seed": 13, "head_seed": 112, "labels": LABELS}))
    tenant = {"x": "A", "y": "B", "y2": "B"}
    srv = Server(eng, m.registry, 3, 128, manager=m)
    hot = [branch["keys"][i] for i in range(len(branch["key_len"])) if branch["key_len"][i] == 3]
    reqs = _requests(3, 9, hot)
    iids = ["x", "y", "x", "y", "x", "y", "x", "y", "x"]
    res = _serve(srv, tenant, iids, reqs, "r")
    assert sorted({r.batch_id for r in res}) == [0, 1, 2]  # 9 requests, max_batch 3
    # bypass oracle: the same answers from retrieve_sequence + higher_stack_forward on the CPU
    tree = oracle.OracleTree(CFG.max_fragment, CFG.hidden_size)
    root = m.versions[0].table
    tree.add_table(0, 0xFFFFFFFF, root["key_len"], root["keys"], root["reps"])
    tree.add_table(v, 0, branch["key_len"], branch["keys"], branch["reps"])
    higher = oracle.generate_higher(CFG)
    seeds = {"x": (11, 111, v), "y": (12, 112, 0)}
    from tests.world import logit_error
    for r, iid, t in zip(res, iids, reqs):
        a, h, ver = seeds[iid]
        w, bb = oracle.generate_head(CFG.hidden_size, LABELS, h)
        s, lab, _ = oracle.infer_one(CFG, higher, tree, ver, t, oracle.generate_adapter(CFG, R, a), R, w, bb)
        assert logit_error(np.float32([r.output.scores]), s[None]) <= 2e-2
    # two instances on the same version and head seed differ only in adapters -> outputs differ
    y = _serve(srv, tenant, ["y", "y2"], [reqs[1], reqs[1]], "d")
    assert y[0].output.scores != y[1].output.scores
    # isolation: A's manage ops never change B's outputs, bit for bit
    before = [r.output.scores for r in _serve(srv, tenant, ["y"] * 4, reqs[:4], "i")]
    m.submit(ManageRequest("update_domain", "A", {"version_id": v, "corpus": _corpus(8, 3, 40, 20, 60)}))
    m.submit(ManageRequest("update_instance", "A", {"instance_id": "x", "adapter_seed": 99}))
    m.submit(ManageRequest("create_instance", "A", {"instance_id": "z", "version_id": 0,
                                                    "adapter_seed": 5, "head_seed": 6}))
    m.submit(ManageRequest("delete_instance", "A", {"instance_id": "z"}))
    after = [r.output.scores for r in _serve(srv, tenant, ["y"] * 4, reqs[:4], "j")]
    assert after == before
    assert m.snapshot_state()["instances"]["x"]["version"] == v + 1
    # save / load on a fresh engine reproduces routing and outputs
    want = _serve(srv, tenant, ["x", "y", "y2"], reqs[:3], "s")
    m.save(str(tmp_path))
    mc = E.model_config(*oracle.astuple(CFG))
    eng2 = E.GpuEngine(mc, E.generate_higher(mc), max_batch=32, max_seq=128, bottleneck=R,
                       max_labels=LABELS, max_tasks=16, max_versions=8)
    m2 = Manager.load(str(tmp_path), eng2, b, min_corpus_tokens=200)
    assert m2.snapshot_state() == m.snapshot_state()
    srv2 = Server(eng2, m2.registry, 3, 128, manager=m2)
    got = _serve(srv2, tenant, ["x", "y", "y2"], reqs[:3], "s")
    assert [r.output.scores for r in got] == [r.output.scores for r in want]
    # delete, then infer against it -> routing error
    m.handle(ManageRequest("delete_instance", "A", {"instance_id": "x"}))
    with pytest.raises(RoutingError):
        srv.enqueue(InferRequest("q", "A", "x", [1, 2, 3]))
    eng2.close()
    eng.close()
    b.close()


@pytest.mark.gpu
def test_gpu_ten_thousand_instances():
    """create_instance x 10,000 under one backbone all succeed; the HBM slot pool
    (here 1,000 tenants' worth) keeps residency within capacity while serving them."""
    n = 10_000
    layer_bytes = (CFG.hidden_size * R * 2 + R + CFG.hidden_size) * 4
    cap = 1000 * CFG.higher_layers * layer_bytes
    eng, b, m = _gpu_world(max_tasks=n, pool_bytes=cap)
    for i in range(n):
        m.submit(ManageRequest("create_instance", f"t{i % 97}", {
            "instance_id": f"i{i}", "version_id": 0, "adapter_seed": i, "head_seed": i % 7}))
    assert m.apply_pending() == n
    assert len(m.snapshot_state()["instances"]) == n
    srv = Server(eng, m.registry, 32, 128, manager=m)
    rng = np.random.default_rng(0)
    for k in range(256):
        i = int(rng.integers(0, n))
        srv.enqueue(InferRequest(f"r{k}", f"t{i % 97}", f"i{i}", list(map(int, rng.integers(0, 300, 12)))))
    assert len(srv.run()) == 256
    st = eng.pool_stats()
    assert st["max_resident_bytes_seen"] <= st["capacity_bytes"] == cap
    eng.close()
    b.close()
