# SPDX-License-Identifier: Apache-2.0
"""bench.py — mixed-tenant hPLM serving throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N --steps K --warmup W] [--config c2] [--mode fine]
    torchrun --nproc-per-node N bench.py --gpus N ...          (tenant-sharded, weak scaling)
    python bench.py --impl reference ...                        (reference CPU path, oracle/_ref)

A step = one mixed-tenant batch (256 requests x 128 tokens per GPU) through the
whole hot path: on-device routing + PLOT retrieval, 6 shared higher layers with
the tenant-grouped adapter GEMMs, per-tenant heads. Rank r serves the tenants
t with t % N == r (own slot pool, replicated shared layers and PLOT tables);
the data path has no collective — torch.distributed is used only for the
barrier and the max-over-ranks of the timings.

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "hBERT-base mixed-tenant req/s at 1/2/4/8 B200; % of bf16 tensor-core peak"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), float(p["bf16_tflops"]), float(p["bf16_tflops_sustained"]), "measured"
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        if os.environ.get("HMI_BENCH_NO_CLOCKS"):  # variance experiments only
            return
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8 or not parts[0].isdigit() or int(parts[0]) != self.gpu:
                continue
            try:
                sm.append(float(parts[1]))
                mx = max(mx, float(parts[2]))
            except ValueError:
                continue
            for n, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def cpu_model() -> str:
    """Host CPU model name and socket count (the CPU arm states its hardware)."""
    try:
        with open("/proc/cpuinfo") as f:
            names = [ln.split(":", 1)[1].strip() for ln in f if ln.startswith("model name")]
        with open("/proc/cpuinfo") as f:
            sockets = {ln.split(":", 1)[1].strip() for ln in f if ln.startswith("physical id")}
        return f"{names[0]} ({len(names)} logical CPUs, {max(len(sockets), 1)} socket(s))"
    except Exception:
        return "unknown"


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist

        global _BACKEND
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        # NCCL needs one GPU per rank; ranks sharing a device (logic check on a small box)
        # or CPU-only runs use gloo. Only the barrier and the timing max go through it.
        _BACKEND = "nccl" if _cuda() and world <= torch.cuda.device_count() else "gloo"
        dist.init_process_group(_BACKEND)
    return world, rank, local


_BACKEND = "gloo"


def _cuda() -> bool:
    import torch

    return torch.cuda.is_available()


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def gather_over_ranks(x: float, world: int) -> list:
    if world == 1:
        return [x]
    import torch
    import torch.distributed as dist

    dev = "cuda" if _BACKEND == "nccl" else "cpu"
    out = [torch.zeros(1, dtype=torch.float64, device=dev) for _ in range(world)]
    dist.all_gather(out, torch.tensor([x], dtype=torch.float64, device=dev))
    return [float(t.item()) for t in out]


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cuda" if _BACKEND == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ---------------------------------------------------------------------------
# reference CPU path (oracle/_ref = the reference compiled from its sources)
# ---------------------------------------------------------------------------
def reference_world(wl, world, tenants):
    import oracle

    if oracle.ref() is None:
        return None
    cfg = oracle.Config(wl.hidden_size, wl.heads, wl.lower_layers, wl.higher_layers, wl.ffn_size,
                        wl.vocab_size, wl.mode, wl.max_fragment, wl.model_seed)
    model = oracle.RefModel(cfg)
    t0 = world.tables[0]
    tree = oracle.RefTree(wl.max_fragment, wl.hidden_size, t0["key_len"], t0["keys"], t0["reps"])
    for t in world.tables[1:]:
        v = tree.add_branch(t["parent"], t["key_len"], t["keys"], t["reps"])
        assert v == t["version"]
    tasks = {int(t): oracle.RefTask(cfg, f"task{t}", wl.r, 1000 + int(t), wl.labels,
                                    2_000_000 + int(t), wl.head_kind) for t in tenants}
    return model, tree, tasks


def run_reference_sample(ref, world, wl, n, seed, threads):
    import oracle

    model, tree, tasks = ref
    inst, toks, lens = world.requests(seed, n, tenants=list(tasks.keys()))
    versions = np.array([world.tenant_version(int(t)) for t in inst], np.uint32)
    t0 = time.perf_counter()
    oracle.ref_infer(model, tree, versions, [tasks[int(t)] for t in inst], toks, lens, wl.labels,
                     threads=threads)
    return time.perf_counter() - t0


def cpu_baseline(wl, world, steps=1, threads=None, sample=None):
    import oracle

    threads = threads or os.cpu_count() or 1
    sample = sample or max(4, threads)
    rng = np.random.default_rng(7)
    tenants = sorted(set(int(x) for x in rng.integers(0, wl.n_tenants, sample)))
    ref = reference_world(wl, world, tenants)
    kind = "reference"
    if ref is None:
        return None
    secs = 0.0
    for s in range(steps):
        secs += run_reference_sample(ref, world, wl, sample, 9000 + s, threads)
    v = steps * sample / secs
    return {"value": v, "unit": "req/s", "cores": threads, "kind": kind, "cpu": cpu_model(),
            "sample": f"{steps}x{sample} {wl.name} requests (seq {wl.seq}) through "
                      f"retrieve_sequence + higher_stack_forward (HMI_KERNELS="
                      f"{oracle.ref().ref_active_kernels().decode()}), {threads} threads"}


def bench_reference(args, wl):
    world_size, rank, _ = dist_setup()
    if rank != 0:
        return
    from paper_2504_17449_b200.workload import World

    world = World(wl)
    threads = os.cpu_count() or 1
    sample = max(2, threads)
    rng = np.random.default_rng(7)
    tenants = sorted(set(int(x) for x in rng.integers(0, wl.n_tenants, 4 * sample)))
    ref = reference_world(wl, world, tenants)
    cfgd = config_dict(wl, args, world_size)
    if ref is None:
        print(json.dumps({"impl": "reference", "unavailable": "reference sources and oracle/_ref both absent"}))
        return
    for s in range(args.warmup):
        run_reference_sample(ref, world, wl, sample, 100 + s, threads)
    secs = 0.0
    for s in range(args.steps):
        secs += run_reference_sample(ref, world, wl, sample, 200 + s, threads)
    v = args.steps * sample / secs
    import oracle

    line = {
        "metric": METRIC, "value": v, "unit": "req/s", "n_gpus": world_size, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * secs / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": cfgd, "impl": "reference",
        "cpu_baseline": {"value": v, "unit": "req/s", "cores": threads, "kind": "reference",
                         "cpu": cpu_model(),
                         "sample": f"each step {sample} requests, {threads} host threads, "
                                   f"HMI_KERNELS={oracle.ref().ref_active_kernels().decode()}"},
        "e2e": {"value": v, "unit": "req/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _union(iv):
    out = []
    for a, b in sorted(iv):
        if out and a <= out[-1][1]:
            out[-1][1] = max(out[-1][1], b)
        else:
            out.append([a, b])
    return out


def _overlap(x, y):
    """Total length of the intersection of two sorted disjoint interval lists."""
    tot, j = 0.0, 0
    for a, b in x:
        while j < len(y) and y[j][1] <= a:
            j += 1
        k = j
        while k < len(y) and y[k][0] < b:
            tot += max(0.0, min(b, y[k][1]) - max(a, y[k][0]))
            k += 1
    return tot


def config_dict(wl, args, world_size):
    return {
        "workload": f"{args.config.upper()} {wl.name}: {wl.n_tenants} tenants, "
                    f"{wl.n_domains} domains{' x ' + str(wl.subdomains) + ' sub-domains' if wl.subdomains else ''}, "
                    f"seq {wl.seq}, batch {wl.batch} per GPU, r={wl.r}, {wl.labels} labels",
        "model": f"{wl.name} ({wl.lower_layers} PLOT + {wl.higher_layers} higher layers, d={wl.hidden_size})",
        "global_batch": wl.batch * world_size,
        "seq_len": wl.seq,
        "parallelism": f"tenant-sharded x{world_size} (no collectives)",
        "pipeline": args.mode,
        "hbm_slot_pool": f"{args.pool_fraction if args.pool_fraction is not None else wl.pool_fraction:.2f}"
                         " of this GPU's tenants",
        "l2": "flushed (256 MiB write) before every timed step",
    }


# ---------------------------------------------------------------------------
# our CUDA path
# ---------------------------------------------------------------------------
def bench_ours(args, wl):
    import torch

    world_size, rank, local = dist_setup()
    # one process per GPU; when more ranks than GPUs are launched (logic check on a
    # single-GPU box) ranks share devices round-robin
    local = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    from paper_2504_17449_b200 import engine as E
    from paper_2504_17449_b200.workload import World

    world = World(wl)
    mode = {"sync": E.MODE_SYNC, "coarse": E.MODE_COARSE, "fine": E.MODE_FINE}[args.mode]
    mc = E.model_config(wl.hidden_size, wl.heads, wl.lower_layers, wl.higher_layers, wl.ffn_size,
                        wl.vocab_size, wl.mode, wl.max_fragment, wl.model_seed)
    higher = E.generate_higher(mc)
    my_tenants = [t for t in range(wl.n_tenants) if t % world_size == rank]
    ref_layer_bytes = (wl.hidden_size * wl.r * 2 + wl.r + wl.hidden_size) * 4
    frac = args.pool_fraction if args.pool_fraction is not None else wl.pool_fraction
    pool_bytes = int(max(wl.batch, frac * len(my_tenants))) * wl.higher_layers * ref_layer_bytes
    eng = E.GpuEngine(mc, higher, device=local, precision=args.precision, max_batch=wl.batch,
                      max_seq=wl.seq, bottleneck=wl.r, max_labels=wl.labels, pipeline_mode=mode,
                      pool_bytes=pool_bytes, max_tasks=wl.n_tenants,
                      max_versions=len(world.tables) + 1)
    for t in world.tables:
        eng.upload_table(t["version"], t["parent"], t["key_len"], t["keys"], t["reps"])
    for t in my_tenants:
        eng.register_task(t, E.generate_adapter(mc, wl.r, 1000 + t))
        w, b = E.generate_head(wl.hidden_size, wl.labels, 2_000_000 + t)
        eng.register_head(t, wl.head_kind, w, b)
        eng.bind_instance(t, world.tenant_version(t), t, t)

    K, W = args.steps, args.warmup
    # W warm-up batches, K timed device-resident batches, K fresh batches for the e2e pass
    # (fresh so a swapping pool sees the same miss rate in both passes)
    # (and, when the pool swaps, K more fresh batches for the StageTrace pass)
    batches = [world.requests(10_000 * (rank + 1) + s, wl.batch, tenants=my_tenants)
               for s in range(W + 3 * K)]
    dev = torch.device("cuda", local)
    d_tok = [torch.from_numpy(b[1].astype(np.int32)).to(dev) for b in batches]
    d_len = [torch.from_numpy(b[2].astype(np.int32)).to(dev) for b in batches]
    d_scores = torch.zeros((wl.batch, wl.labels), dtype=torch.float32, device=dev)
    d_labels = torch.zeros((wl.batch,), dtype=torch.int32, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.ExternalStream(eng.stream, device=dev)
    torch.cuda.synchronize()

    def run_device(i):
        inst, _, lens = batches[i]
        eng.infer_batch_device(inst, d_tok[i].data_ptr(), wl.seq, d_len[i].data_ptr(),
                               int(lens.max()), d_scores.data_ptr(), d_labels.data_ptr())

    clocks = ClockSampler(local)
    clocks.start()  # sampled from the warm-up through the timed region
    # warm-up: one pass over every tenant of this rank (fills the slot pool up to its
    # capacity), then W ordinary batches
    for c in range(0, len(my_tenants), wl.batch):
        chunk = np.array(my_tenants[c:c + wl.batch], np.uint32)
        _, toks, lens = world.requests(77 + c, len(chunk), tenants=chunk)
        eng.infer_batch(chunk, toks, lens)
    for i in range(W):
        run_device(i)
    eng.synchronize()
    for i in range(W):  # second pass so the pool is warm for the steady state
        run_device(i)
    eng.synchronize()

    # ---- timed: inputs resident in HBM, L2 flushed before each step
    c0 = E.engine_counters(eng)
    p0 = eng.pool_stats()
    barrier(world_size)
    torch.cuda.synchronize()
    evs = []
    with torch.cuda.stream(stream):
        for k in range(K):
            flush.zero_()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            run_device(W + k)
            b.record(stream)
            evs.append((a, b))
    eng.synchronize()
    torch.cuda.synchronize()
    barrier(world_size)
    clk = clocks.stop()
    c1 = E.engine_counters(eng)
    p1 = eng.pool_stats()
    local_ms = sum(a.elapsed_time(b) for a, b in evs)
    max_ms = max_over_ranks(local_ms, world_size)
    value = world_size * wl.batch * K / (max_ms / 1e3)
    if args.quick:  # timed region only (used under ncu)
        if rank == 0:
            print(json.dumps({"metric": METRIC, "value": value, "unit": "req/s", "quick": True,
                              "ms_per_step": max_ms / K}), flush=True)
        eng.close()
        return

    # ---- e2e: public host-buffer API (hmi_gpu_submit_batch / hmi_gpu_wait_batch, two batches
    # in flight as a serving loop runs them): every step's H2D of tokens / lengths / instance
    # ids from host memory and D2H of scores / labels lie inside the timed region
    barrier(world_size)
    torch.cuda.synchronize()
    for i in range(min(W, 2)):
        inst, toks, lens = batches[i]
        eng.infer_batch(inst, toks, lens)
    t0 = time.perf_counter()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record(stream)
    depth = int(os.environ.get("HMI_E2E_DEPTH", "2"))  # batches in flight (3 and 4 measured no better)
    inflight = []
    for k in range(K):
        inst, toks, lens = batches[W + K + k]
        inflight.append(eng.submit_batch(inst, toks, lens))
        if len(inflight) >= depth:
            eng.wait_batch(inflight.pop(0))
    for t in inflight:
        eng.wait_batch(t)
    b.record(stream)
    torch.cuda.synchronize()
    e2e_ms = max(a.elapsed_time(b), 1e3 * (time.perf_counter() - t0))
    e2e_ms = max_over_ranks(e2e_ms, world_size)
    e2e = world_size * wl.batch * K / (e2e_ms / 1e3)
    h2d = wl.batch * (wl.seq * 4 + 4 + 4)          # tokens + lens + instance ids
    d2h = wl.batch * (wl.labels * 4 + 4)           # scores + labels

    # ---- per-kernel device time (events around every launch) for the roofline
    eng.profile(True)
    for k in range(K):
        with torch.cuda.stream(stream):
            flush.zero_()
        run_device(W + k)
    eng.synchronize()
    prof = eng.profile_read()
    eng.profile(False)

    # ---- adapter swap (pool below all of this rank's tenants): bytes copied per timed step,
    # and from a StageTrace of K more device-resident batches the io (H2D) busy time and the
    # share of it that overlaps compute
    swap = None
    if frac < 1.0:
        eng.trace(True)
        for k in range(K):
            run_device(W + 2 * K + k)
        eng.synchronize()
        recs = eng.stage_trace()
        eng.trace(False)
        io = _union([(r["start_ms"], r["end_ms"]) for r in recs if r["worker"] == "io"])
        comp = _union([(r["start_ms"], r["end_ms"]) for r in recs if r["worker"] == "compute"])
        io_busy = sum(b - a for a, b in io)
        comp_busy = sum(b - a for a, b in comp)
        span = comp[-1][1] - comp[0][0] if comp else 0.0
        copied = (p1["bytes_copied"] - p0["bytes_copied"]) / K
        swap = {"bytes_copied_per_step": copied,
                "loads_per_step": (p1["loads"] - p0["loads"]) / K,
                "transfers_per_step": (c1["adapter_copies"] - c0["adapter_copies"]) / K,
                "io_busy_ms_per_step": io_busy / K, "compute_busy_ms_per_step": comp_busy / K,
                "compute_idle_ms_per_step": (span - comp_busy) / K,
                "io_hidden_frac": _overlap(io, comp) / io_busy if io_busy > 0 else 1.0,
                "hide_threshold_gbps": copied / (max_ms / K * 1e-3) / 1e9}

    # ---- concurrent host -> HBM copy rate per rank (all ranks at once after a barrier), from
    # NUMA-local pinned memory as the adapter store: whether PCIe or the socket link caps the
    # swap of C4 / C5 on a full box
    barrier(world_size)
    h2d_rate = gather_over_ranks(E.h2d_probe(eng), world_size)
    numa = gather_over_ranks(float(-1 if c1["numa_node"] is None else c1["numa_node"]), world_size)

    hbm, peak_burst, peak_sust, peak_src = peaks()
    T = wl.batch * wl.seq
    d, f, r = wl.hidden_size, wl.ffn_size, wl.r
    flops = {"gemm_qkv": 2 * T * d * 3 * d, "gemm_oproj": 2 * T * d * d, "gemm_ffn1": 2 * T * d * f,
             "gemm_ffn2": 2 * T * f * d, "adapter_down": 2 * T * d * r, "adapter_up": 2 * T * r * d}
    step_ms = sum(v[0] for k, v in prof.items() if k not in ("step",)) / max(K, 1)
    dom = max(flops, key=lambda k: prof[k][0])
    ms_dom = prof[dom][0] / max(prof[dom][1], 1)
    achieved = flops[dom] / (ms_dom * 1e-3) / 1e12
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as fh:
            traffic = json.load(fh).get("kernels", {}).get(dom, {}).get("dram_bytes")
    except Exception:
        pass
    kernels = {k: {"ms_per_launch": v[0] / max(v[1], 1), "launches": v[1],
                   "share": v[0] / max(step_ms * K, 1e-9)} for k, v in prof.items() if v[1]}
    for k in flops:
        if k in kernels:
            kernels[k]["tflops"] = flops[k] / (kernels[k]["ms_per_launch"] * 1e-3) / 1e12

    line = {
        "metric": METRIC,
        "value": value,
        "unit": "req/s",
        "n_gpus": world_size,
        "steps": K,
        "warmup": W,
        "ms_per_step": max_ms / K,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "fp16 operands, fp32 accumulate" if args.precision == 0 else "bf16 operands, fp32 accumulate",
        "data": "synthetic (seeded generate_model / adapters / heads, synthetic PLOT tables)",
        "config": config_dict(wl, args, world_size),
        "e2e": {"value": e2e, "unit": "req/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "l2": "not flushed: back-to-back serving loop, two batches in flight (the device-"
                      "timed value flushes L2 before every step)"},
        "gpu_launches": int(c1["launches"] - c0["launches"]),
        "roofline": {
            "bound": "tensor", "kernel": dom, "achieved": achieved, "peak": peak_sust,
            "unit": "TFLOP/s", "frac": achieved / peak_sust, "traffic": traffic,
            "peak_source": f"{peak_src} bf16_tflops_sustained (kernel timed inside a long step)",
            "frac_of_burst": achieved / peak_burst,
            "step_tensor_frac": value / world_size * wl.flops_per_request() / 1e12 / peak_burst,
            "flops_per_request": wl.flops_per_request(),
        },
        "kernels": kernels,
        "clocks": clk,
        "pool": eng.pool_stats(),
        "h2d_gbps_per_rank": [round(x, 2) for x in h2d_rate],
        "swap": swap,
        "pinned_numa_node_per_rank": [int(x) for x in numa],
    }
    if rank == 0 and world_size == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(wl, world)
    if rank == 0:
        print(json.dumps(line), flush=True)
    eng.close()


def bench_generate(args, wl):
    """C3: mixed-tenant greedy generation (prompt wl.seq + wl.gen_tokens tokens) through
    hmi_gpu_generate; one shared vocabulary lm head. A step = one batch of wl.batch
    requests from prompt to last token. Reported beside the C2 headline, not instead."""
    import torch

    world_size, rank, local = dist_setup()
    local = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    from paper_2504_17449_b200 import engine as E
    from paper_2504_17449_b200.workload import World

    world = World(wl)
    mc = E.model_config(wl.hidden_size, wl.heads, wl.lower_layers, wl.higher_layers, wl.ffn_size,
                        wl.vocab_size, wl.mode, wl.max_fragment, wl.model_seed)
    higher = E.generate_higher(mc)
    my_tenants = [t for t in range(wl.n_tenants) if t % world_size == rank]
    eng = E.GpuEngine(mc, higher, device=local, precision=args.precision, max_batch=wl.batch,
                      max_seq=wl.seq, bottleneck=wl.r, max_labels=8,
                      pipeline_mode=E.MODE_FINE, max_tasks=wl.n_tenants,
                      max_versions=len(world.tables) + 1, max_new_tokens=wl.gen_tokens)
    for t in world.tables:
        eng.upload_table(t["version"], t["parent"], t["key_len"], t["keys"], t["reps"])
    w, b = E.generate_head(wl.hidden_size, wl.labels, 2_000_000)
    eng.register_head(0, wl.head_kind, w, b)
    for t in my_tenants:
        eng.register_task(t, E.generate_adapter(mc, wl.r, 1000 + t))
        eng.bind_instance(t, world.tenant_version(t), t, 0)
    K, W = args.steps, args.warmup
    batches = [world.requests(10_000 * (rank + 1) + s, wl.batch, tenants=my_tenants)
               for s in range(W + K)]
    for c in range(0, len(my_tenants), wl.batch):  # fill the slot pool
        chunk = np.array(my_tenants[c:c + wl.batch], np.uint32)
        _, toks, lens = world.requests(77 + c, len(chunk), tenants=chunk)
        eng.infer_batch(chunk, toks, lens)
    for i in range(W):
        eng.generate(batches[i][0], batches[i][1], batches[i][2], wl.gen_tokens)
    stream = torch.cuda.ExternalStream(eng.stream, device=torch.device("cuda", local))
    c0 = E.engine_counters(eng)
    barrier(world_size)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    a = torch.cuda.Event(enable_timing=True)
    b_ = torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for k in range(K):
        inst, toks, lens = batches[W + k]
        eng.generate(inst, toks, lens, wl.gen_tokens)
    b_.record(stream)
    torch.cuda.synchronize()
    ms = max(a.elapsed_time(b_), 1e3 * (time.perf_counter() - t0))
    ms = max_over_ranks(ms, world_size)
    c1 = E.engine_counters(eng)
    value = world_size * wl.batch * K / (ms / 1e3)
    hbm, peak_burst, _, _ = peaks()

    # ---- decode-step roofline (HBM-bound): the same K batches generating one
    # token (prompt forward + lm head) time the prefill; the remaining gen_tokens - 1 single-row
    # steps take the difference. Algorithmic bytes of one step at this batch: every shared
    # weight, the lm head, each distinct tenant's adapter slots, the KV cache up to the step's
    # context, and the f32 logits written and read once.
    torch.cuda.synchronize()
    a1 = torch.cuda.Event(enable_timing=True)
    b1 = torch.cuda.Event(enable_timing=True)
    a1.record(stream)
    for k in range(K):
        inst, toks, lens = batches[W + k]
        eng.generate(inst, toks, lens, 1)
    b1.record(stream)
    torch.cuda.synchronize()
    ms1 = max_over_ranks(a1.elapsed_time(b1), world_size)
    step_ms = (ms - ms1) / K / (wl.gen_tokens - 1)
    d, f, r, L, V, B = wl.hidden_size, wl.ffn_size, wl.r, wl.higher_layers, wl.labels, wl.batch
    w_shared = L * (4 * d * d + 2 * d * f) * 2
    w_lm = V * d * 2
    tenants = float(np.mean([len(set(batches[W + k][0].tolist())) for k in range(K)]))
    slot = (2 * r * d) * 2 + (r + d) * 4
    w_adapt = tenants * L * slot
    ctx_mean = float(np.mean([batches[W + k][2].mean() for k in range(K)])) + wl.gen_tokens / 2
    kv = B * ctx_mean * L * 2 * d * 2
    logits = 2 * B * V * 4
    step_bytes = w_shared + w_lm + w_adapt + kv + logits
    roof = {"bound": "hbm", "kernel": "decode step (all kernels of one generated token)",
            "achieved": step_bytes / (step_ms * 1e-3) / 1e9, "peak": hbm, "unit": "GB/s",
            "frac": step_bytes / (step_ms * 1e-3) / 1e9 / hbm, "traffic": None,
            "step_ms": step_ms, "prefill_ms": ms1 / K,
            "bytes_per_step": {"shared_weights": w_shared, "lm_head": w_lm,
                               "adapters": w_adapt, "kv_cache": kv, "logits": logits,
                               "total": step_bytes, "distinct_tenants": tenants,
                               "mean_context": ctx_mean}}
    # ---- per-class device time (CUDA events around every launch: a separate profile pass; the
    # events cost the programmatic-launch overlap, so the sum exceeds the timed batch)
    eng.profile(True)
    for k in range(K):
        inst, toks, lens = batches[W + k]
        eng.generate(inst, toks, lens, wl.gen_tokens)
    torch.cuda.synchronize()
    prof = eng.profile_read()
    eng.profile(False)
    kernels = {c: {"ms_per_batch": v[0] / K, "launches_per_batch": v[1] / K}
               for c, v in prof.items() if v[1]}
    line = {
        "metric": f"{wl.name} mixed-tenant generated requests/s (prompt {wl.seq} + {wl.gen_tokens} tokens)",
        "value": value, "unit": "req/s", "n_gpus": world_size, "steps": K, "warmup": W,
        "ms_per_step": ms / K, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "fp16 operands, fp32 accumulate", "data": "synthetic",
        "config": config_dict(wl, args, world_size),
        "tokens_per_s": value * wl.gen_tokens,
        "e2e": {"value": value, "unit": "req/s", "h2d_bytes_per_step": wl.batch * (wl.seq * 4 + 8),
                "d2h_bytes_per_step": wl.batch * wl.gen_tokens * 8},
        "gpu_launches": int(c1["launches"] - c0["launches"]),
        "roofline": roof,
        "kernels": kernels,
        "tensor_frac": value / world_size * wl.generate_flops_per_request() / 1e12 / peak_burst,
        "flops_per_request": wl.generate_flops_per_request(),
        "note": "host API timed (hmi_gpu_generate, synchronous per batch); a side config, the "
                "headline is C2",
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    eng.close()


def bench_plot(args):
    """GPU PLOT builder: lower_stack_forward of the C2 root table's
    keys (the vocabulary uni-gram backstop + every 2/3-gram of the root corpus, build_root's key
    set, table.cpp:29-58) through hmi_plot_forward, host keys in / host f32 reps out. A step =
    the whole root table. Side measurement; the headline is C2 serving."""
    import torch

    world_size, rank, local = dist_setup()
    if rank != 0:
        return
    torch.cuda.set_device(local)
    from paper_2504_17449_b200 import engine as E
    from paper_2504_17449_b200 import plot
    from paper_2504_17449_b200.workload import CONFIGS, World

    wl = CONFIGS["c2"]
    world = World(wl)
    root = world.tables[0]
    key_len, keys = root["key_len"], root["keys"]
    rows = int(key_len.sum())
    mc = E.model_config(wl.hidden_size, wl.heads, wl.lower_layers, wl.higher_layers, wl.ffn_size,
                        wl.vocab_size, wl.mode, wl.max_fragment, wl.model_seed)
    b = plot.GpuPlotBuilder(mc, max_rows=32768)
    for _ in range(args.warmup):
        b.forward(key_len[:4096], keys[:4096])
    clocks = ClockSampler(local)
    clocks.start()
    ms0, _ = b.stats()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        reps = b.forward(key_len, keys)
    secs = time.perf_counter() - t0
    ms1, _ = b.stats()
    clk = clocks.stop()
    d, f = wl.hidden_size, wl.ffn_size
    flops_row = 2 * (4 * d * d + 2 * d * f) * wl.lower_layers
    value = args.steps * rows / ((ms1 - ms0) / 1e3)   # device time of the GPU passes
    e2e = args.steps * rows / secs                    # host keys in -> host f32 reps out
    _, peak_burst, peak_sust, peak_src = peaks()
    achieved = value * flops_row / 1e12
    line = {
        "metric": "PLOT build: lower-stack rows/s (C2 root table: 30,522 uni-grams + corpus 2/3-grams)",
        "value": value, "unit": "rows/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * secs / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "fp16 operands, fp32 accumulate", "data": "synthetic corpus",
        "config": {"workload": f"hBERT-base lower stack ({wl.lower_layers} layers, d={d}), "
                               f"{len(key_len)} keys / {rows} rows per step",
                   "l2": "inputs (rows x d activations per layer) exceed L2"},
        "e2e": {"value": e2e, "unit": "rows/s", "h2d_bytes_per_step": int(keys.nbytes + key_len.nbytes),
                "d2h_bytes_per_step": int(reps.nbytes)},
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak_sust, "unit": "TFLOP/s",
                     "frac": achieved / peak_sust, "traffic": None,
                     "peak_source": f"{peak_src} bf16_tflops_sustained; all lower-stack kernels of the step",
                     "flops_per_row": flops_row},
        "clocks": clk,
    }
    if not args.no_cpu_baseline:
        import oracle
        from concurrent.futures import ThreadPoolExecutor

        cfg = oracle.Config(wl.hidden_size, wl.heads, wl.lower_layers, wl.higher_layers,
                            wl.ffn_size, wl.vocab_size, wl.mode, wl.max_fragment, wl.model_seed)
        m = oracle.generate_model(cfg, lower=True)
        threads = os.cpu_count() or 1
        sample = list(range(0, len(key_len), max(1, len(key_len) // (4 * threads))))[:4 * threads]
        t0 = time.perf_counter()
        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(lambda i: oracle.lower_forward(cfg, m, keys[i, :key_len[i]]), sample))
        cs = time.perf_counter() - t0
        line["cpu_baseline"] = {"value": int(key_len[sample].sum()) / cs, "unit": "rows/s",
                                "cores": threads, "kind": "port", "cpu": cpu_model(),
                                "sample": f"{len(sample)} root-table fragments through the C oracle's "
                                          f"lower_stack_forward (bit-exact to the reference's scalar "
                                          f"kernels), {threads} threads"}
    print(json.dumps(line), flush=True)
    b.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2")
    ap.add_argument("--mode", default="fine", choices=["sync", "coarse", "fine"])
    ap.add_argument("--precision", type=int, default=0)
    ap.add_argument("--pool-fraction", type=float, default=None,
                    help="HBM slot pool as a fraction of this rank's tenants (C4 sweep)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--quick", action="store_true", help="timed device region only (for ncu)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    from paper_2504_17449_b200.workload import CONFIGS

    if args.config == "plot":
        bench_plot(args)
        return
    wl = CONFIGS[args.config]
    if args.impl == "reference":
        bench_reference(args, wl)
    elif wl.gen_tokens:
        bench_generate(args, wl)
    else:
        bench_ours(args, wl)


if __name__ == "__main__":
    main()
