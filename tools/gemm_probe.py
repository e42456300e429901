# SPDX-License-Identifier: Apache-2.0
"""Runs one K1 GEMM probe launch pair (for ncu): python tools/gemm_probe.py M N K bn epi"""
import sys

import numpy as np

sys.path.insert(0, ".")
from tests.test_gemm_gpu import _probe  # noqa: E402

M, N, K, bn, epi = (int(x) for x in sys.argv[1:6])
rng = np.random.default_rng(0)
a = rng.standard_normal((M, K)).astype(np.float16)
b = rng.uniform(-0.05, 0.05, (1, N, K)).astype(np.float16)
r0 = rng.standard_normal((M, N)).astype(np.float16) if epi & 2 else None
out, ms = _probe(a, b, np.zeros((1, N), np.float32), res0=r0, epi=epi, bn=bn)
print(f"{M}x{N}x{K} bn={bn} epi={epi}: {ms:.4f} ms {2.0 * M * N * K / ms / 1e9:.0f} TFLOP/s")
