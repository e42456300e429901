// SPDX-License-Identifier: Apache-2.0
//
// Kernels of the GPU PLOT builder (plot_builder.cpp): the lower stack's embedding and the
// attention core over PLOT fragments (n-grams of <= max_fragment tokens).
//
//   lower_stack_forward (proj/src/transformer/model.cpp:96-118): h[i] = token_emb[t_i] +
//   position_emb[i] (fragment-local positions), then the lower layers (layer_forward without an
//   adapter, model.cpp:84-94). The projections / FFN run on the tcgen05 GEMM; only the
//   fragment-sized attention (model.cpp:39-74, keys j < len or j <= i) is specific here.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <cstdint>

#include "plot_builder.hpp"

namespace hmi_b200 {

namespace {

template <bool kBf16>
__device__ __forceinline__ float2 ld2(const uint16_t* p) {
  const uint32_t w = *reinterpret_cast<const uint32_t*>(p);
  if constexpr (kBf16) {
    return __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w));
  } else {
    return __half22float2(*reinterpret_cast<const __half2*>(&w));
  }
}

template <bool kBf16>
__device__ __forceinline__ void st2(uint16_t* p, float a, float b) {
  uint32_t w;
  if constexpr (kBf16) {
    const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    w = *reinterpret_cast<const uint32_t*>(&h);
  } else {
    const __half2 h = __floats2half2_rn(a, b);
    w = *reinterpret_cast<const uint32_t*>(&h);
  }
  *reinterpret_cast<uint32_t*>(p) = w;
}

// one block per row: h16[r] = token_emb[key] + position_emb[pos]; rows >= n * k are zero
template <bool kBf16>
__global__ void plot_embed_kernel(const float* __restrict__ tok_emb,
                                  const float* __restrict__ pos_emb,
                                  const uint32_t* __restrict__ keys, int ngram, int k, int n,
                                  int d, uint16_t* __restrict__ h16) {
  const int r = blockIdx.x;
  const int f = r / k, i = r - (r / k) * k;
  uint16_t* out = h16 + static_cast<size_t>(r) * d;
  if (f >= n) {
    for (int c = 2 * threadIdx.x; c < d; c += 2 * blockDim.x) st2<kBf16>(out + c, 0.f, 0.f);
    return;
  }
  const uint32_t t = __ldg(&keys[static_cast<size_t>(f) * ngram + i]);
  const float* te = tok_emb + static_cast<size_t>(t) * d;
  const float* pe = pos_emb + static_cast<size_t>(i) * d;
  for (int c = 2 * threadIdx.x; c < d; c += 2 * blockDim.x) {
    const float2 a = *reinterpret_cast<const float2*>(te + c);
    const float2 b = *reinterpret_cast<const float2*>(pe + c);
    st2<kBf16>(out + c, a.x + b.x, a.y + b.y);
  }
}

// one warp per (fragment, head); lane owns head dims 2*lane, 2*lane+1 (head size 64)
template <bool kBf16>
__global__ void plot_attention_kernel(const uint16_t* __restrict__ qkv, uint16_t* __restrict__ ctx,
                                      int k, int n, int heads, int d, int causal, float scale) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= n * heads) return;
  const int f = warp / heads, h = warp - (warp / heads) * heads;
  const size_t ld = static_cast<size_t>(3) * d;
  const uint16_t* base = qkv + static_cast<size_t>(f) * k * ld + h * 64 + 2 * lane;
  float2 kk[kMaxFragment], vv[kMaxFragment];
#pragma unroll
  for (int j = 0; j < kMaxFragment; ++j) {
    if (j < k) {
      kk[j] = ld2<kBf16>(base + j * ld + d);
      vv[j] = ld2<kBf16>(base + j * ld + 2 * d);
    }
  }
  for (int i = 0; i < k; ++i) {
    const float2 q = ld2<kBf16>(base + i * ld);
    const int lim = causal ? i + 1 : k;
    float s[kMaxFragment];
    float mx = -INFINITY;
#pragma unroll
    for (int j = 0; j < kMaxFragment; ++j) {
      if (j < lim) {
        float p = q.x * kk[j].x + q.y * kk[j].y;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) p += __shfl_xor_sync(0xffffffffu, p, o);
        s[j] = p * scale;
        mx = fmaxf(mx, s[j]);
      }
    }
    float sum = 0.f, ox = 0.f, oy = 0.f;
#pragma unroll
    for (int j = 0; j < kMaxFragment; ++j) {
      if (j < lim) {
        const float e = __expf(s[j] - mx);
        sum += e;
        ox += e * vv[j].x;
        oy += e * vv[j].y;
      }
    }
    const float inv = 1.f / sum;
    st2<kBf16>(ctx + static_cast<size_t>(f * k + i) * d + h * 64 + 2 * lane, ox * inv, oy * inv);
  }
}

}  // namespace

void launch_plot_embed(const float* tok_emb, const float* pos_emb, const uint32_t* keys, int ngram,
                       int k, int n, int rows, int d, void* h16, int precision,
                       cudaStream_t stream) {
  if (rows <= 0) return;
  if (precision == 1) {
    plot_embed_kernel<true><<<rows, 128, 0, stream>>>(tok_emb, pos_emb, keys, ngram, k, n, d,
                                                      static_cast<uint16_t*>(h16));
  } else {
    plot_embed_kernel<false><<<rows, 128, 0, stream>>>(tok_emb, pos_emb, keys, ngram, k, n, d,
                                                       static_cast<uint16_t*>(h16));
  }
  HMI_CUDA(cudaGetLastError());
}

void launch_plot_attention(const void* qkv, void* ctx, int k, int n, int heads, int d, int causal,
                           int precision, cudaStream_t stream) {
  if (n <= 0) return;
  HMI_CHECK(d == heads * 64 && k >= 1 && k <= kMaxFragment, HMI_CONFIG_ERROR,
            "plot attention: head size 64, fragment length <= 5");
  const float scale = 1.0f / sqrtf(static_cast<float>(d / heads));
  const int warps = n * heads;
  const int blocks = (warps + 7) / 8;
  if (precision == 1) {
    plot_attention_kernel<true><<<blocks, 256, 0, stream>>>(
        static_cast<const uint16_t*>(qkv), static_cast<uint16_t*>(ctx), k, n, heads, d, causal, scale);
  } else {
    plot_attention_kernel<false><<<blocks, 256, 0, stream>>>(
        static_cast<const uint16_t*>(qkv), static_cast<uint16_t*>(ctx), k, n, heads, d, causal, scale);
  }
  HMI_CUDA(cudaGetLastError());
}

}  // namespace hmi_b200
