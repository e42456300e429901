# SPDX-License-Identifier: Apache-2.0
"""Adapter-slot H2D transfer rates: python tools/copy_probe.py"""
import ctypes
import sys

sys.path.insert(0, ".")
from paper_2504_17449_b200 import _native  # noqa: E402

L = _native.lib()
for n, b in ((600, 200704), (100, 1204224)):
    for mode, name in ((0, "one copy"), (1, "n memcpyAsync"), (3, "zero-copy 16"),
                       (4, "zero-copy 32"), (5, "zero-copy 64")):
        g = ctypes.c_double(0)
        m = min(mode, 3)
        ctas = {3: 16, 4: 32, 5: 64}.get(mode, 0)
        rc = L.hmi_gpu_copy_probe(0, n, b, m, ctas, ctypes.byref(g))
        print(f"{n} x {b // 1024} KB {name:18s}: {g.value:6.1f} GB/s rc={rc}", flush=True)
