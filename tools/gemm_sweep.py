# SPDX-License-Identifier: Apache-2.0
"""K1 shapes of the C2 step: our tcgen05 GEMM (1-CTA / cta_group::2, each N tile) against
torch.matmul (cuBLAS) on the same fp16 operands.  python tools/gemm_sweep.py [--ncu]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from tests.test_gemm_gpu import _probe  # noqa: E402

SHAPES = {"qkv": (32768, 2304, 768, 0), "oproj": (32768, 768, 768, 0),
          "ffn1": (32768, 3072, 768, 1), "ffn2": (32768, 768, 3072, 0)}
ncu = "--ncu" in sys.argv
rng = np.random.default_rng(0)
for name, (M, N, K, epi) in SHAPES.items():
    a = rng.standard_normal((M, K)).astype(np.float16)
    b = rng.uniform(-0.05, 0.05, (1, N, K)).astype(np.float16)
    bias = np.zeros((1, N), np.float32)
    ref = None
    for bn in (128, 192, 256):
        if N % bn:
            continue
        for c2 in (0, 1):
            best = 1e9
            for _ in range(1 if ncu else 3):
                out, ms = _probe(a, b, bias, epi=epi | (256 if c2 else 0), bn=bn)
                best = min(best, ms)
            if ref is None:
                ref = out
            ok = np.array_equal(out, ref)
            print(f"ours {name:6s} {M}x{N}x{K} bn={bn} cta2={c2}: {best * 1e3:7.1f} us "
                  f"{2.0 * M * N * K / best / 1e9:6.0f} TFLOP/s  same-as-first={ok}", flush=True)
    if ncu:
        continue
    ta = torch.from_numpy(a).cuda()
    tb = torch.from_numpy(b[0]).cuda()
    for _ in range(3):
        ta @ tb.T
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(20):
        ta @ tb.T
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(f"cublas {name:6s} {M}x{N}x{K}: {ms * 1e3:7.1f} us {2.0 * M * N * K / ms / 1e9:6.0f} TFLOP/s",
          flush=True)
