# SPDX-License-Identifier: Apache-2.0
"""Decode-shape GEMMs (M = 256): the K1 kernel per N tile / CTA form vs cuBLAS (torch.matmul).
python tools/decode_gemm_probe.py"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from tests.test_gemm_gpu import _probe  # noqa: E402

rng = np.random.default_rng(0)
for (N, K) in ((2304, 768), (768, 768), (3072, 768), (768, 1024), (768, 3072)):
    M = 256
    a = rng.standard_normal((M, K)).astype(np.float16)
    b = rng.uniform(-0.05, 0.05, (1, N, K)).astype(np.float16)
    res = []
    for bn, flag in ((64, 0), (128, 0), (128, 256), (256, 256)):
        if N % bn:
            continue
        ms = min(_probe(a, b, np.zeros((1, N), np.float32), epi=flag, bn=bn)[1] for _ in range(5))
        res.append(f"bn{bn}{'p' if flag else ''}={ms * 1e3:.1f}us")
    ta = torch.from_numpy(a).cuda()
    tb = torch.from_numpy(b[0]).cuda()
    for _ in range(10):
        torch.matmul(ta, tb.t())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(50):
        torch.matmul(ta, tb.t())
    e1.record()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(50):
            torch.matmul(ta, tb.t())
    g.replay()
    torch.cuda.synchronize()
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2.record()
    g.replay()
    e3.record()
    torch.cuda.synchronize()
    wbytes = N * K * 2
    print(f"M={M} N={N} K={K} ({wbytes / 1e6:.1f} MB weights): " + " ".join(res) +
          f"  cublas={e0.elapsed_time(e1) / 50 * 1e3:.1f}us graph={e2.elapsed_time(e3) / 50 * 1e3:.1f}us")
