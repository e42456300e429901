# SPDX-License-Identifier: Apache-2.0
"""Pinned-host -> HBM bandwidth vs the NUMA node the pinned pages land on."""
import os
import sys

import torch

dev = torch.device("cuda", 0)
bus = torch.cuda.get_device_properties(0).pci_bus_id if hasattr(torch.cuda.get_device_properties(0), "pci_bus_id") else None
import ctypes
cudart = ctypes.CDLL("libcudart.so") if False else None
busid = ctypes.create_string_buffer(64)
lib = ctypes.CDLL(torch.__file__.replace("__init__.py", "lib/libc10_cuda.so"))
try:
    rt = ctypes.CDLL("libcudart.so.12")
except OSError:
    import glob
    rt = ctypes.CDLL(glob.glob("/usr/local/cuda/lib64/libcudart.so*")[0])
rt.cudaDeviceGetPCIBusId(busid, 64, 0)
b = busid.value.decode().lower()
print("gpu bus", b)
base = f"/sys/bus/pci/devices/{b}"
if not os.path.exists(base):
    base = f"/sys/bus/pci/devices/{b.replace('00000000:', '0000:')}"
for f in ("numa_node", "local_cpulist"):
    try:
        print(f, open(os.path.join(base, f)).read().strip())
    except OSError as e:
        print(f, "n/a", e)
print("nodes", sorted(os.listdir("/sys/devices/system/node")) if os.path.exists("/sys/devices/system/node") else "n/a")
for n in sorted(d for d in os.listdir("/sys/devices/system/node") if d.startswith("node")):
    print(n, open(f"/sys/devices/system/node/{n}/cpulist").read().strip())
print("affinity", sorted(os.sched_getaffinity(0))[:8], "...", len(os.sched_getaffinity(0)))


def parse(lst):
    out = []
    for part in lst.split(","):
        if "-" in part:
            a, c = part.split("-")
            out += list(range(int(a), int(c) + 1))
        elif part:
            out.append(int(part))
    return out


def bw():
    piece = 200704 * 512
    h = torch.empty(piece, dtype=torch.uint8).pin_memory()
    h.fill_(1)
    d = torch.empty(piece, dtype=torch.uint8, device=dev)
    best = 0
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        d.copy_(h, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        best = max(best, piece / e0.elapsed_time(e1) / 1e6)
    return best


allc = sorted(os.sched_getaffinity(0))
print(f"default affinity: {bw():.1f} GB/s")
for n in sorted(d for d in os.listdir("/sys/devices/system/node") if d.startswith("node")):
    cpus = [c for c in parse(open(f"/sys/devices/system/node/{n}/cpulist").read().strip()) if c in allc]
    if not cpus:
        continue
    os.sched_setaffinity(0, cpus)
    print(f"pinned pages allocated from {n}: {bw():.1f} GB/s")
    os.sched_setaffinity(0, allc)
