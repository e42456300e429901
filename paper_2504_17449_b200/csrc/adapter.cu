// SPDX-License-Identifier: Apache-2.0
//
// Adapter fold (registration time). The reference applies each tenant's adapter to the
// attention output a = ctx.Wo + bo (proj/src/transformer/model.cpp:13-24, :75, :87-89):
//
//   mid = ReLU(a.Wd + bd)          out = mid.Wu + bu + a
//
// a.Wd + bd = ctx.(Wo.Wd) + (bo.Wd + bd), so the down projection can read ctx directly.
// Registration stores, in each (task, layer) slot, Wc^T = (Wo.Wd)^T [r_pad][d] 16-bit and
// bc = bo.Wd + bd in place of Wd^T and bd. On the hot path the tenant-grouped GEMM
// mid = ReLU(ctx.Wc + bc) then needs no O projection before it, and the up projection becomes
// extra K blocks of the O projection itself (gemm_tcgen05.cuh, kEpiExt):
//
//   y1 = [ctx | mid] . [Wo ; Wu] + bo + bu + LN2_{l-1}(y2)
//
// Everything downstream of the slot (swap pool, peer export, decode) sees bytes of the same
// size and layout. Wc is computed in f32 from the slot's 16-bit Wd^T (the bytes the hot
// path multiplies today) and the layer's f32 Wo, then rounded once.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <cstdint>

#include "adapter.hpp"

namespace hmi_b200 {

namespace {

constexpr int kFoldThreads = 256;
constexpr int kTile = 64;   // 64 (j) x 64 (k) outputs per CTA
constexpr int kChunk = 32;  // reduction (i) chunk staged in shared memory

__device__ __forceinline__ float ld16f(const uint16_t* p, int bf16) {
  const uint16_t u = *p;
  return bf16 ? __uint_as_float(static_cast<uint32_t>(u) << 16) : __half2float(__ushort_as_half(u));
}

__device__ __forceinline__ uint16_t st16f(float v, int bf16) {
  return bf16 ? __bfloat16_as_ushort(__float2bfloat16_rn(v)) : __half_as_ushort(__float2half_rn(v));
}

// grid (d / 64, r_pad / 64, slot images); slot image s is (task s / L, layer s % L).
//   out Wc^T[j][k] = sum_i Wd^T[j][i] * Wo[k][i]        Wo row-major [in k][out i]
//   out bc[j]      = bd[j] + sum_i bo[i] * Wd^T[j][i]   (CTAs with blockIdx.x == 0)
__global__ void __launch_bounds__(kFoldThreads) fold_kernel(const uint8_t* __restrict__ in,
                                                            uint8_t* __restrict__ out,
                                                            const float* __restrict__ wo,
                                                            const float* __restrict__ bo, int L,
                                                            int d, int r_pad, size_t slot_bytes,
                                                            size_t off_bd, int bf16) {
  __shared__ float As[kChunk][kTile + 1];  // Wd^T chunk, [i][j]
  __shared__ float Bs[kChunk][kTile + 1];  // Wo chunk, [i][k]
  const int s = blockIdx.z;
  const int layer = s % L;
  const int j0 = blockIdx.y * kTile, k0 = blockIdx.x * kTile;
  const uint16_t* wdt = reinterpret_cast<const uint16_t*>(in + static_cast<size_t>(s) * slot_bytes);
  const float* wol = wo + static_cast<size_t>(layer) * d * d;
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
  float acc[4][4] = {};
  for (int i0 = 0; i0 < d; i0 += kChunk) {
#pragma unroll
    for (int q = 0; q < (kTile * kChunk) / kFoldThreads; ++q) {
      const int e = tid + q * kFoldThreads;
      const int row = e / kChunk, ii = e % kChunk;  // consecutive threads: consecutive i
      As[ii][row] = ld16f(wdt + static_cast<size_t>(j0 + row) * d + i0 + ii, bf16);
      Bs[ii][row] = wol[static_cast<size_t>(k0 + row) * d + i0 + ii];
    }
    __syncthreads();
#pragma unroll 8
    for (int ii = 0; ii < kChunk; ++ii) {
      float a[4], b[4];
#pragma unroll
      for (int m = 0; m < 4; ++m) a[m] = As[ii][ty + 16 * m];
#pragma unroll
      for (int n = 0; n < 4; ++n) b[n] = Bs[ii][tx + 16 * n];
#pragma unroll
      for (int m = 0; m < 4; ++m)
#pragma unroll
        for (int n = 0; n < 4; ++n) acc[m][n] = fmaf(a[m], b[n], acc[m][n]);
    }
    __syncthreads();
  }
  uint16_t* wct = reinterpret_cast<uint16_t*>(out + static_cast<size_t>(s) * slot_bytes);
#pragma unroll
  for (int m = 0; m < 4; ++m)
#pragma unroll
    for (int n = 0; n < 4; ++n)
      wct[static_cast<size_t>(j0 + ty + 16 * m) * d + k0 + tx + 16 * n] = st16f(acc[m][n], bf16);
  if (blockIdx.x == 0) {
    // bias: 4 threads per output j, strided over i, then a 4-lane reduction
    const float* bd = reinterpret_cast<const float*>(in + static_cast<size_t>(s) * slot_bytes + off_bd);
    float* bc = reinterpret_cast<float*>(out + static_cast<size_t>(s) * slot_bytes + off_bd);
    const float* bol = bo + static_cast<size_t>(layer) * d;
    const int j = j0 + (tid >> 2), p = tid & 3;
    float sum = 0.f;
    for (int i = p; i < d; i += 4) sum = fmaf(bol[i], ld16f(wdt + static_cast<size_t>(j) * d + i, bf16), sum);
    sum += __shfl_xor_sync(0xffffffffu, sum, 1);
    sum += __shfl_xor_sync(0xffffffffu, sum, 2);
    if (p == 0) bc[j] = bd[j] + sum;
  }
}

}  // namespace

void launch_adapter_fold(const uint8_t* in, uint8_t* out, int n_images, const float* wo,
                         const float* bo, int L, int d, int r_pad, size_t slot_bytes,
                         size_t off_bd, int precision, cudaStream_t stream) {
  if (n_images <= 0) return;
  HMI_CHECK(d % kTile == 0 && r_pad % kTile == 0, HMI_CONFIG_ERROR,
            "adapter fold: hidden size and padded bottleneck must be multiples of 64");
  fold_kernel<<<dim3(d / kTile, r_pad / kTile, n_images), kFoldThreads, 0, stream>>>(
      in, out, wo, bo, L, d, r_pad, slot_bytes, off_bd, precision == 1 ? 1 : 0);
  HMI_CUDA(cudaGetLastError());
}

}  // namespace hmi_b200
