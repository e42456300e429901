// SPDX-License-Identifier: Apache-2.0
//
// K3 — fused multi-head attention core per (request, head, 64-query block).
//
// Restates the score / softmax / PV loops of attention() (proj/src/transformer/
// model.cpp:39-74): s_j = (q_i . k_j) / sqrt(dh) over keys j < limit, with
// limit = valid_len (encoder) or i + 1 (causal); keys outside the window are
// never read (model.cpp:48-51), softmax is max-subtracted, ctx = sum p_j v_j / sum p_j.
// The Q/K/V projections and the output projection are K1 GEMMs around this kernel.
//
// Input : qkv [T x 3d] 16-bit (q | k | v column blocks), request b owns rows [b*S, b*S+S)
// Output: ctx [T x d] 16-bit
// dh = 64. One CTA = 8 warps = 128 query rows (K/V read once per (request, head)); K/V streamed through smem in 64-key
// blocks with an online softmax (fp32 statistics), tensor-core mma.sync m16n8k16.
// Memory bound at hBERT shapes (reads 3 x 16 KB, writes 16 KB per (request, head)).
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <cstdint>

#include "kernels.hpp"
#include "sm100.cuh"

namespace hmi_b200 {

namespace {

constexpr int kDh = 64;
constexpr int kQB = 128;   // query rows per CTA (8 warps x 16)
constexpr int kKB = 64;    // keys per block
constexpr int kPad = 72;   // smem row stride in 16-bit elements (144 B: conflict-free ldmatrix)

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(smem))),
               "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(p))));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(p))));
}

template <bool kBf16>
__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0,
                                         uint32_t b1) {
  if constexpr (kBf16) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
  } else {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
  }
}

template <bool kBf16>
__device__ __forceinline__ uint32_t pack2(float x, float y) {
  if constexpr (kBf16) {
    __nv_bfloat162 h = __floats2bfloat162_rn(x, y);
    return *reinterpret_cast<uint32_t*>(&h);
  } else {
    __half2 h = __floats2half2_rn(x, y);
    return *reinterpret_cast<uint32_t*>(&h);
  }
}

template <bool kBf16>
__global__ void __launch_bounds__(256, 2) attention_kernel(const uint16_t* __restrict__ qkv,
                                                        uint16_t* __restrict__ ctx,
                                                        const int* __restrict__ lens, int S,
                                                        int d, int causal, float scale_log2) {
  extern __shared__ __align__(128) uint16_t att_smem[];
  uint16_t* sQ = att_smem;                                   // [kQB][kPad]
  uint16_t* const sK0 = sQ + kQB * kPad;       // [2][kKB][kPad]
  uint16_t* const sV0 = sK0 + 2 * kKB * kPad;   // [2][kKB][kPad]

  const int qb = blockIdx.x, head = blockIdx.y, b = blockIdx.z;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int valid = lens[b];
  const long long row0 = static_cast<long long>(b) * S;
  const int ld = 3 * d;
  const uint16_t* gq = qkv + (row0 + qb * kQB) * ld + head * kDh;
  const uint16_t* gk = qkv + row0 * ld + d + head * kDh;
  const uint16_t* gv = qkv + row0 * ld + 2 * d + head * kDh;

  // number of key blocks this CTA must visit
  int nkb;
  if (causal) {
    nkb = (qb + 1) * (kQB / kKB);
  } else {
    nkb = (valid + kKB - 1) / kKB;
  }
  if (nkb < 1) nkb = 1;

  auto load_tile = [&](uint16_t* dst, const uint16_t* src) {  // 64 rows x 128 B
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int c = tid + i * 256;  // 512 chunks of 16 B
      const int r = c >> 3, cc = c & 7;
      cp_async16(dst + r * kPad + cc * 8, src + static_cast<long long>(r) * ld + cc * 8);
    }
  };
  load_tile(sQ, gq);
  load_tile(sQ + 64 * kPad, gq + 64ll * ld);
  load_tile(sK0, gk);
  load_tile(sV0, gv);
  cp_async_commit();

  const int g = lane >> 2, tq = lane & 3;
  const int qrow_a = qb * kQB + warp * 16 + g;  // rows held by this thread: qrow_a, qrow_a + 8
  const int lim_a = causal ? qrow_a + 1 : valid;
  const int lim_b = causal ? qrow_a + 9 : valid;

  float m_a = -INFINITY, m_b = -INFINITY, l_a = 0.f, l_b = 0.f;
  float o[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  uint32_t qf[4][4];

  for (int kb = 0; kb < nkb; ++kb) {
    if (kb + 1 < nkb) {
      load_tile(sK0 + ((kb + 1) & 1) * kKB * kPad, gk + static_cast<long long>((kb + 1) * kKB) * ld);
      load_tile(sV0 + ((kb + 1) & 1) * kKB * kPad, gv + static_cast<long long>((kb + 1) * kKB) * ld);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    if (kb == 0) {
#pragma unroll
      for (int ks = 0; ks < 4; ++ks)
        ldsm_x4(qf[ks], sQ + (warp * 16 + (lane & 15)) * kPad + ks * 16 + (lane >> 4) * 8);
    }
    const uint16_t* K = sK0 + (kb & 1) * kKB * kPad;
    const uint16_t* V = sV0 + (kb & 1) * kKB * kPad;

    // S = Q K^T : 16 x 64 per warp
    float s[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i) s[i][0] = s[i][1] = s[i][2] = s[i][3] = 0.f;
#pragma unroll
    for (int np = 0; np < 4; ++np) {  // pairs of 8-key n tiles
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        uint32_t bf[4];
        ldsm_x4(bf, K + (np * 16 + (lane & 7) + ((lane >> 4) << 3)) * kPad + ks * 16 +
                        ((lane >> 3) & 1) * 8);
        mma16816<kBf16>(s[2 * np], qf[ks], bf[0], bf[1]);
        mma16816<kBf16>(s[2 * np + 1], qf[ks], bf[2], bf[3]);
      }
    }
    // mask + online softmax (base-2 with pre-scaled logits)
    float mx_a = m_a, mx_b = m_b;
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      const int key = kb * kKB + nt * 8 + 2 * tq;
      s[nt][0] = key < lim_a ? s[nt][0] * scale_log2 : -INFINITY;
      s[nt][1] = key + 1 < lim_a ? s[nt][1] * scale_log2 : -INFINITY;
      s[nt][2] = key < lim_b ? s[nt][2] * scale_log2 : -INFINITY;
      s[nt][3] = key + 1 < lim_b ? s[nt][3] * scale_log2 : -INFINITY;
      mx_a = fmaxf(mx_a, fmaxf(s[nt][0], s[nt][1]));
      mx_b = fmaxf(mx_b, fmaxf(s[nt][2], s[nt][3]));
    }
    mx_a = fmaxf(mx_a, __shfl_xor_sync(0xffffffffu, mx_a, 1));
    mx_a = fmaxf(mx_a, __shfl_xor_sync(0xffffffffu, mx_a, 2));
    mx_b = fmaxf(mx_b, __shfl_xor_sync(0xffffffffu, mx_b, 1));
    mx_b = fmaxf(mx_b, __shfl_xor_sync(0xffffffffu, mx_b, 2));
    const float base_a = mx_a == -INFINITY ? 0.f : mx_a;
    const float base_b = mx_b == -INFINITY ? 0.f : mx_b;
    const float corr_a = exp2f(m_a - base_a), corr_b = exp2f(m_b - base_b);
    m_a = mx_a;
    m_b = mx_b;
    float sum_a = 0.f, sum_b = 0.f;
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      s[nt][0] = exp2f(s[nt][0] - base_a);
      s[nt][1] = exp2f(s[nt][1] - base_a);
      s[nt][2] = exp2f(s[nt][2] - base_b);
      s[nt][3] = exp2f(s[nt][3] - base_b);
      sum_a += s[nt][0] + s[nt][1];
      sum_b += s[nt][2] + s[nt][3];
    }
    l_a = l_a * corr_a + sum_a;
    l_b = l_b * corr_b + sum_b;
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      o[nt][0] *= corr_a; o[nt][1] *= corr_a;
      o[nt][2] *= corr_b; o[nt][3] *= corr_b;
    }
    // O += P V
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {  // 16 keys per step
      uint32_t pa[4];
      pa[0] = pack2<kBf16>(s[2 * ks][0], s[2 * ks][1]);
      pa[1] = pack2<kBf16>(s[2 * ks][2], s[2 * ks][3]);
      pa[2] = pack2<kBf16>(s[2 * ks + 1][0], s[2 * ks + 1][1]);
      pa[3] = pack2<kBf16>(s[2 * ks + 1][2], s[2 * ks + 1][3]);
#pragma unroll
      for (int np = 0; np < 4; ++np) {  // pairs of 8-wide dh tiles
        uint32_t bf[4];
        ldsm_x4_t(bf, V + (ks * 16 + (lane & 7) + ((lane >> 3) & 1) * 8) * kPad + np * 16 +
                          (lane >> 4) * 8);
        mma16816<kBf16>(o[2 * np], pa, bf[0], bf[1]);
        mma16816<kBf16>(o[2 * np + 1], pa, bf[2], bf[3]);
      }
    }
    __syncthreads();  // buffer (kb & 1) is overwritten by the load issued next iteration
  }
  l_a += __shfl_xor_sync(0xffffffffu, l_a, 1);
  l_a += __shfl_xor_sync(0xffffffffu, l_a, 2);
  l_b += __shfl_xor_sync(0xffffffffu, l_b, 1);
  l_b += __shfl_xor_sync(0xffffffffu, l_b, 2);
  const float inv_a = l_a > 0.f ? 1.f / l_a : 0.f;
  const float inv_b = l_b > 0.f ? 1.f / l_b : 0.f;
  uint16_t* out_a = ctx + (row0 + qrow_a) * d + head * kDh;
  uint16_t* out_b = out_a + 8ll * d;
#pragma unroll
  for (int nt = 0; nt < 8; ++nt) {
    const int col = nt * 8 + 2 * tq;
    *reinterpret_cast<uint32_t*>(out_a + col) = pack2<kBf16>(o[nt][0] * inv_a, o[nt][1] * inv_a);
    *reinterpret_cast<uint32_t*>(out_b + col) = pack2<kBf16>(o[nt][2] * inv_b, o[nt][3] * inv_b);
  }
}

}  // namespace

AttnPlan make_attention_plan(const void* qkv, void* ctx, int max_rows, int d, int precision) {
  AttnPlan p;
  const CUtensorMapDataType t16 =
      precision == 1 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  p.map_qkv = make_tmap_2d(qkv, t16, 3ull * d, max_rows, 3ull * d * 2, 64, 128,
                           CU_TENSOR_MAP_SWIZZLE_128B);
  p.map_ctx = make_tmap_2d(ctx, t16, d, max_rows, static_cast<uint64_t>(d) * 2, 64, 128,
                           CU_TENSOR_MAP_SWIZZLE_128B);
  p.d = d;
  p.precision = precision;
  return p;
}

void launch_attention(const void* qkv, void* ctx, const int* lens, int n_req, int S, int d,
                      int heads, int causal, int precision, cudaStream_t stream) {
  HMI_CHECK(d == heads * kDh, HMI_CONFIG_ERROR, "attention: head width must be 64");
  HMI_CHECK(S % kQB == 0, HMI_DIMENSION_ERROR, "attention: padded length must be a multiple of 128");
  if (n_req <= 0) return;
  const float scale_log2 = 1.4426950408889634f / sqrtf(static_cast<float>(kDh));
  dim3 grid(S / kQB, heads, n_req);
  const int smem = (kQB + 4 * kKB) * kPad * 2;
  static bool configured[2] = {false, false};
  if (!configured[precision == 1]) {
    if (precision == 1) {
      HMI_CUDA(cudaFuncSetAttribute(attention_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    } else {
      HMI_CUDA(cudaFuncSetAttribute(attention_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    }
    configured[precision == 1] = true;
  }
  if (precision == 1) {
    attention_kernel<true><<<grid, 256, smem, stream>>>(static_cast<const uint16_t*>(qkv),
                                                     static_cast<uint16_t*>(ctx), lens, S, d,
                                                     causal, scale_log2);
  } else {
    attention_kernel<false><<<grid, 256, smem, stream>>>(static_cast<const uint16_t*>(qkv),
                                                      static_cast<uint16_t*>(ctx), lens, S, d,
                                                      causal, scale_log2);
  }
  HMI_CUDA(cudaGetLastError());
}

}  // namespace hmi_b200
