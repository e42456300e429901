# SPDX-License-Identifier: Apache-2.0
"""K1/K2 tcgen05 GEMM vs a plain fp32 reference of the same op.

The fp32 reference consumes exactly the 16-bit operands the kernel sees, so
the only difference is accumulation order (fp32 in TMEM vs numpy fp32/f64).
"""
import ctypes

import numpy as np
import pytest

from paper_2504_17449_b200 import _native

pytestmark = pytest.mark.gpu


def _probe(a, b, bias, tile_slot=None, res0=None, res1=None, epi=0, bn=256, precision=0):
    M, K = a.shape
    G, N, K2 = b.shape
    assert K == K2
    out_f32 = bool(epi & 8)
    out = np.zeros((M, N), dtype=np.float32 if out_f32 else np.uint16)
    ms = ctypes.c_float(0)

    def p(x, t):
        return None if x is None else np.ascontiguousarray(x).ctypes.data_as(ctypes.POINTER(t))

    a16 = np.ascontiguousarray(a.view(np.uint16))
    b16 = np.ascontiguousarray(b.view(np.uint16))
    r0 = None if res0 is None else np.ascontiguousarray(res0.view(np.uint16))
    r1 = None if res1 is None else np.ascontiguousarray(res1.view(np.uint16))
    ts = None if tile_slot is None else np.ascontiguousarray(tile_slot.astype(np.int32))
    bias = np.ascontiguousarray(bias.astype(np.float32))
    st = _native.lib().hmi_gpu_gemm_probe(
        0, M, N, K, G,
        p(a16, ctypes.c_uint16), p(b16, ctypes.c_uint16), p(bias, ctypes.c_float),
        p(ts, ctypes.c_int32), p(r0, ctypes.c_uint16), p(r1, ctypes.c_uint16),
        epi, bn, precision, out.ctypes.data_as(ctypes.c_void_p), ctypes.byref(ms))
    assert st == 0, _native.last_error()
    if not out_f32:
        out = out.view(np.float16).astype(np.float32)
    return out, ms.value


def _ref(a, b, bias, tile_slot, res0=None, res1=None, relu=False):
    M = a.shape[0]
    a32 = a.astype(np.float64)
    out = np.empty((M, b.shape[1]), dtype=np.float64)
    slots = np.zeros(M // 128, dtype=np.int64) if tile_slot is None else tile_slot
    for t in range(M // 128):
        g = slots[t]
        out[t * 128:(t + 1) * 128] = a32[t * 128:(t + 1) * 128] @ b[g].astype(np.float64).T + bias[g]
    if res0 is not None:
        out += res0.astype(np.float64)
    if res1 is not None:
        out += res1.astype(np.float64)
    if relu:
        out = np.maximum(out, 0)
    return out


@pytest.mark.parametrize("M,N,K,bn", [(128, 256, 64, 256), (256, 768, 768, 192),
                                       (1024, 2304, 768, 256), (512, 768, 3072, 192),
                                       (384, 128, 256, 128), (256, 64, 768, 64)])
def test_gemm_shared_bias(M, N, K, bn):
    rng = np.random.default_rng(M + N + K)
    a = rng.standard_normal((M, K)).astype(np.float16)
    b = (rng.uniform(-0.05, 0.05, (1, N, K))).astype(np.float16)
    bias = rng.uniform(-0.05, 0.05, (1, N)).astype(np.float32)
    out, _ = _probe(a, b, bias, bn=bn)
    ref = _ref(a, b, bias, None)
    err = np.abs(out - ref).max() / np.abs(ref).max()
    assert err < 2e-3, err


@pytest.mark.parametrize("M,N,K,bn,epi", [(256, 256, 64, 256, 0), (384, 768, 768, 192, 0),
                                           (1024, 2304, 768, 256, 1), (512, 768, 3072, 192, 2 | 8),
                                           (640, 3072, 768, 256, 1), (256, 128, 128, 128, 8)])
def test_gemm_cta_pair(M, N, K, bn, epi):
    """cta_group::2 kernel (UMMA M=256 over a CTA pair, B split across the pair);
    odd M-tile counts exercise the idle half of the last pair."""
    rng = np.random.default_rng(M * 7 + N)
    a = rng.standard_normal((M, K)).astype(np.float16)
    b = rng.uniform(-0.05, 0.05, (1, N, K)).astype(np.float16)
    bias = rng.uniform(-0.05, 0.05, (1, N)).astype(np.float32)
    r0 = rng.standard_normal((M, N)).astype(np.float16) if epi & 2 else None
    out, _ = _probe(a, b, bias, res0=r0, epi=epi | 256, bn=bn)
    ref = _ref(a, b, bias, None, r0, relu=bool(epi & 1))
    err = np.abs(out - ref).max() / np.abs(ref).max()
    assert err < 2e-3, err


def test_gemm_cta_pair_throughput():
    rng = np.random.default_rng(6)
    res = {}
    for name, (M, N, K, bn) in {"qkv": (32768, 2304, 768, 256), "ffn1": (32768, 3072, 768, 256),
                                "ffn2": (32768, 768, 3072, 192)}.items():
        a = rng.standard_normal((M, K)).astype(np.float16)
        b = rng.uniform(-0.05, 0.05, (1, N, K)).astype(np.float16)
        bias = np.zeros((1, N), np.float32)
        _, ms1 = _probe(a, b, bias, bn=bn)
        out, ms2 = _probe(a, b, bias, bn=bn, epi=256)
        res[name] = (2.0 * M * N * K / (ms1 * 1e-3) / 1e12, 2.0 * M * N * K / (ms2 * 1e-3) / 1e12)
        ref = a[:256].astype(np.float64) @ b[0].astype(np.float64).T
        assert np.abs(out[:256] - ref).max() / np.abs(ref).max() < 2e-3
    print("TFLOP/s 1-CTA vs 2-CTA:", {k: (round(x), round(y)) for k, (x, y) in res.items()})


def test_gemm_relu_f16():
    rng = np.random.default_rng(1)
    M, N, K = 512, 3072, 768
    a = rng.standard_normal((M, K)).astype(np.float16)
    b = rng.uniform(-0.05, 0.05, (1, N, K)).astype(np.float16)
    bias = rng.uniform(-0.05, 0.05, (1, N)).astype(np.float32)
    out, _ = _probe(a, b, bias, epi=1, bn=256)
    ref = _ref(a, b, bias, None, relu=True)
    assert (out >= 0).all()
    assert np.abs(out - ref).max() / np.abs(ref).max() < 2e-3


def test_gemm_grouped_residual_f32():
    """Tenant-grouped mode: each 128-row tile gathers its own B group."""
    rng = np.random.default_rng(2)
    M, N, K, G = 1024, 768, 64, 5
    a = rng.standard_normal((M, K)).astype(np.float16)
    b = rng.uniform(-0.05, 0.05, (G, N, K)).astype(np.float16)
    bias = rng.uniform(-0.05, 0.05, (G, N)).astype(np.float32)
    slots = rng.integers(0, G, M // 128)
    r0 = rng.standard_normal((M, N)).astype(np.float16)
    r1 = rng.standard_normal((M, N)).astype(np.float16)
    out, _ = _probe(a, b, bias, tile_slot=slots, res0=r0, res1=r1, epi=4 | 8, bn=256)
    ref = _ref(a, b, bias, slots, r0, r1)
    assert np.abs(out - ref).max() < 1e-4 * np.abs(ref).max() + 1e-5


def test_gemm_grouped_down_relu():
    rng = np.random.default_rng(3)
    M, N, K, G = 2048, 64, 768, 7
    a = rng.standard_normal((M, K)).astype(np.float16)
    b = rng.uniform(-0.05, 0.05, (G, N, K)).astype(np.float16)
    bias = rng.uniform(-0.05, 0.05, (G, N)).astype(np.float32)
    slots = rng.integers(0, G, M // 128)
    out, _ = _probe(a, b, bias, tile_slot=slots, epi=1, bn=64)
    ref = _ref(a, b, bias, slots, relu=True)
    assert np.abs(out - ref).max() / np.abs(ref).max() < 2e-3


def test_gemm_bf16_operands():
    import torch

    rng = np.random.default_rng(4)
    M, N, K = 256, 512, 512
    a = torch.from_numpy(rng.standard_normal((M, K)).astype(np.float32)).bfloat16()
    b = torch.from_numpy(rng.uniform(-0.05, 0.05, (1, N, K)).astype(np.float32)).bfloat16()
    bias = rng.uniform(-0.05, 0.05, (1, N)).astype(np.float32)
    out, _ = _probe(a.view(torch.int16).numpy().view(np.uint16),
                    b.view(torch.int16).numpy().view(np.uint16), bias, bn=256, epi=8,
                    precision=1)
    ref = a.double().numpy() @ b[0].double().numpy().T + bias[0]
    assert np.abs(out - ref).max() / np.abs(ref).max() < 1e-4


def test_gemm_throughput_qkv_shape():
    """hBERT-base QKV shape at batch 256 x seq 128: report TFLOP/s (sanity floor only)."""
    rng = np.random.default_rng(5)
    M, N, K = 32768, 2304, 768
    a = rng.standard_normal((M, K)).astype(np.float16)
    b = rng.uniform(-0.05, 0.05, (1, N, K)).astype(np.float16)
    bias = np.zeros((1, N), np.float32)
    out, ms = _probe(a, b, bias, bn=256)
    tflops = 2.0 * M * N * K / (ms * 1e-3) / 1e12
    print(f"QKV gemm {M}x{N}x{K}: {ms:.3f} ms, {tflops:.1f} TFLOP/s")
    ref = a[:256].astype(np.float64) @ b[0].astype(np.float64).T
    assert np.abs(out[:256] - ref).max() / np.abs(ref).max() < 2e-3
    assert tflops > 100


@pytest.mark.parametrize("M,N,K,bn,epi", [(32768, 768, 3072, 256, 2), (32768, 768, 768, 256, 0),
                                           (5120, 768, 768, 192, 8), (20480, 256, 256, 128, 1)])
def test_gemm_cta_pair_wave_tail_split_bit_identical(M, N, K, bn, epi):
    """The pair kernel's last partial wave runs as narrower N sub-tiles (MMA N = BN/2..BN/4);
    every output element keeps its K order, so results are bit-identical to whole tiles."""
    rng = np.random.default_rng(M + N + K)
    a = rng.standard_normal((M, K)).astype(np.float16)
    b = rng.uniform(-0.05, 0.05, (1, N, K)).astype(np.float16)
    bias = rng.uniform(-0.1, 0.1, (1, N)).astype(np.float32)
    r0 = rng.standard_normal((M, N)).astype(np.float16) if epi & 2 else None
    split, _ = _probe(a, b, bias, res0=r0, epi=epi | 256, bn=bn)
    whole, _ = _probe(a, b, bias, res0=r0, epi=epi | 256 | 8192, bn=bn)
    assert np.array_equal(split, whole)
    for rows in (slice(0, 256), slice(M - 256, M)):  # first wave and the split tail
        ref = a[rows].astype(np.float64) @ b[0].astype(np.float64).T + bias[0]
        if epi & 2:
            ref += r0[rows]
        if epi & 1:
            ref = np.maximum(ref, 0)
        assert np.abs(split[rows] - ref).max() / np.abs(ref).max() < 2e-3


# decode-step GEMMs: K-split clusters reduced through DSMEM (gemm_dec.cu). `cfg` = (bn, ks)
# forced, or None for the plan's own choice; ks = 3 / 6 split the tile's rows unevenly
@pytest.mark.parametrize("M,N,K,epi,cfg", [
    (256, 2304, 768, 0, None), (256, 768, 768, 0, None), (256, 3072, 768, 1, None),
    (256, 768, 3072, 2 | 8, None), (128, 2304, 768, 0, None), (256, 768, 768, 8, (64, 2)),
    (256, 2304, 768, 0, (128, 3)), (256, 3072, 768, 1, (256, 6)), (128, 768, 3072, 2 | 8, (64, 8)),
    (384, 1024, 1024, 1, (128, 4))])
def test_decode_gemm_ksplit(M, N, K, epi, cfg):
    rng = np.random.default_rng(M + 3 * N + K)
    a = rng.standard_normal((M, K)).astype(np.float16)
    b = rng.uniform(-0.05, 0.05, (1, N, K)).astype(np.float16)
    bias = rng.uniform(-0.05, 0.05, (1, N)).astype(np.float32)
    r0 = rng.standard_normal((M, N)).astype(np.float16) if epi & 2 else None
    bn = 0 if cfg is None else (cfg[1] << 16) | cfg[0]
    out, _ = _probe(a, b, bias, res0=r0, epi=epi | 16384, bn=bn)
    ref = _ref(a, b, bias, None, r0, relu=bool(epi & 1))
    err = np.abs(out - ref).max() / np.abs(ref).max()
    assert err < 2e-3, err
    again, _ = _probe(a, b, bias, res0=r0, epi=epi | 16384, bn=bn)
    assert np.array_equal(out, again)  # fixed rank order: run-to-run identical


def test_decode_gemm_bf16():
    rng = np.random.default_rng(5)
    M, N, K = 256, 2304, 768
    a32 = rng.standard_normal((M, K)).astype(np.float32)
    b32 = rng.uniform(-0.05, 0.05, (1, N, K)).astype(np.float32)

    def bf16(x):  # round to nearest even on the top 16 bits
        u = x.view(np.uint32).astype(np.uint64)
        u = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
        return u

    a16, b16 = bf16(a32), bf16(b32)
    bias = np.zeros((1, N), np.float32)
    out = np.zeros((M, N), np.float32)
    ms = ctypes.c_float(0)
    st = _native.lib().hmi_gpu_gemm_probe(
        0, M, N, K, 1, a16.ctypes.data_as(ctypes.POINTER(ctypes.c_uint16)),
        b16.ctypes.data_as(ctypes.POINTER(ctypes.c_uint16)),
        bias.ctypes.data_as(ctypes.POINTER(ctypes.c_float)), None, None, None, 8 | 16384, 0, 1,
        out.ctypes.data_as(ctypes.c_void_p), ctypes.byref(ms))
    assert st == 0, _native.last_error()
    up = lambda u: (u.astype(np.uint32) << 16).view(np.float32).astype(np.float64)  # noqa: E731
    ref = up(a16) @ up(b16)[0].T
    assert np.abs(out - ref).max() / np.abs(ref).max() < 2e-3


def test_decode_gemm_no_fit_is_config_error():
    """K / 64 = 17 has no split with at most 16 K blocks per CTA: the decode plan refuses with a
    configuration error (the engine then serves that GEMM with the persistent K1 plan)."""
    rng = np.random.default_rng(9)
    M, N, K = 128, 256, 64 * 17
    a = rng.standard_normal((M, K)).astype(np.float16)
    b = rng.uniform(-0.05, 0.05, (1, N, K)).astype(np.float16)
    bias = np.zeros((1, N), np.float32)
    out = np.zeros((M, N), np.uint16)
    ms = ctypes.c_float(0)
    st = _native.lib().hmi_gpu_gemm_probe(
        0, M, N, K, 1, a.view(np.uint16).ctypes.data_as(ctypes.POINTER(ctypes.c_uint16)),
        b.view(np.uint16).ctypes.data_as(ctypes.POINTER(ctypes.c_uint16)),
        bias.ctypes.data_as(ctypes.POINTER(ctypes.c_float)), None, None, None, 16384, 0, 0,
        out.ctypes.data_as(ctypes.c_void_p), ctypes.byref(ms))
    assert st == _native.ConfigError.code, (st, _native.last_error())
    out2, _ = _probe(a, b, bias, bn=64)  # the K1 kernel serves the same shape
    ref = _ref(a, b, bias, None)
    assert np.abs(out2 - ref).max() / np.abs(ref).max() < 2e-3
