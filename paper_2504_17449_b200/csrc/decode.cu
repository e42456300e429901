// SPDX-License-Identifier: Apache-2.0
//
// Causal (hGPT) generation: the wide lm head and the single-row decode step.
//
// The reference has no decode loop (SPEC.md:188 lists caching as a non-goal);
// greedy generation here is defined as repeated causal forwards, token t+1 =
// argmax of apply_head(lm_logits) at row valid_len - 1 (model.cpp:151-168,
// first max wins, :122-128) of the sequence extended by token t. In causal mode
// row i reads only keys j <= i (model.cpp:48-51) and PLOT rows of the window
// ending at i (retrieval.cpp:92-99), so earlier rows never change and their
// keys / values are cached: one new row per request per step.
//
//   lm_gather_kernel       final row (valid_len - 1) of each request, LayerNorm'd
//                          (f64, ops.cpp:92-116) when the stack leaves it pre-norm;
//                          f32 copy for rescoring, 16-bit copy as the GEMM operand
//   (tcgen05 GEMM)         logits = h . W_lm + b over the padded vocabulary
//   lm_argmax_kernel       top-8 candidates of the 16-bit-operand logits, rescored
//                          in f64 from the f32 row and the f32 head weights; first
//                          max of the rescored values; appends the token
//   attn_decode_kernel     one query row per (request, head) against the cached
//                          keys (prefill rows + generated rows); appends its k, v
//   adapter_rows_ln_kernel per-row tenant adapter (each decode row may belong to a
//                          different tenant: the slot is gathered per row), skip
//                          and residual adds, LayerNorm1 (model.cpp:13-24, 87-92)
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <cstdint>

#include "decode.hpp"
#include "sm100.cuh"

namespace hmi_b200 {

namespace {

__device__ __forceinline__ float ld16(const uint16_t* p, long long i, int bf16) {
  const uint16_t u = p[i];
  if (bf16) return __uint_as_float(static_cast<uint32_t>(u) << 16);
  return __half2float(__ushort_as_half(u));
}

__device__ __forceinline__ uint16_t st16(float v, int bf16) {
  if (bf16) return __bfloat16_as_ushort(__float2bfloat16_rn(v));
  return __half_as_ushort(__float2half_rn(v));
}

// unpack 8 16-bit values of a uint4 into floats
__device__ __forceinline__ void unpack8(const uint4& u, float* f, int bf16) {
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    if (bf16) {
      f[2 * i] = __uint_as_float(w[i] << 16);
      f[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
    } else {
      const __half2 h = *reinterpret_cast<const __half2*>(&w[i]);
      const float2 t = __half22float2(h);
      f[2 * i] = t.x;
      f[2 * i + 1] = t.y;
    }
  }
}

template <typename T>
__device__ __forceinline__ T block_sum_t(T v, T* scratch) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  __syncthreads();
  if (lane == 0) scratch[warp] = v;
  __syncthreads();
  T t = 0;
  for (int w = 0; w < nw; ++w) t += scratch[w];
  __syncthreads();
  return t;
}

__device__ __forceinline__ float block_max_f(float v, float* scratch) {
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  __syncthreads();
  if (lane == 0) scratch[warp] = v;
  __syncthreads();
  float t = -INFINITY;
  for (int w = 0; w < nw; ++w) t = fmaxf(t, scratch[w]);
  __syncthreads();
  return t;
}

// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) lm_gather_kernel(const uint16_t* __restrict__ y16,
                                                        const float* __restrict__ h32,
                                                        const float* __restrict__ g,
                                                        const float* __restrict__ be,
                                                        const int* __restrict__ lens, int S, int d,
                                                        int bf16, float* __restrict__ out32,
                                                        uint16_t* __restrict__ out16) {
  extern __shared__ double xs[];
  __shared__ double red[32];
  const int b = blockIdx.x;
  const long long rbase = (static_cast<long long>(b) * S + lens[b] - 1) * d;
  if (y16) {
    double s1 = 0.0;
    for (int j = threadIdx.x; j < d; j += blockDim.x) {
      xs[j] = ld16(y16, rbase + j, bf16);
      s1 += xs[j];
    }
    const double mean = block_sum_t(s1, red) / d;
    double s2 = 0.0;
    for (int j = threadIdx.x; j < d; j += blockDim.x) {
      const double t = xs[j] - mean;
      s2 += t * t;
    }
    const double inv = 1.0 / sqrt(block_sum_t(s2, red) / d + 1e-5);
    for (int j = threadIdx.x; j < d; j += blockDim.x) {
      const float v = static_cast<float>((xs[j] - mean) * inv * g[j] + be[j]);
      out32[static_cast<long long>(b) * d + j] = v;
      out16[static_cast<long long>(b) * d + j] = st16(v, bf16);
    }
  } else {
    for (int j = threadIdx.x; j < d; j += blockDim.x) {
      const float v = h32[rbase + j];
      out32[static_cast<long long>(b) * d + j] = v;
      out16[static_cast<long long>(b) * d + j] = st16(v, bf16);
    }
  }
}

// ---------------------------------------------------------------------------
constexpr int kTopK = 8;
constexpr int kArgThreads = 256;

__global__ void __launch_bounds__(kArgThreads) lm_argmax_kernel(LmArgmaxArgs A) {
  __shared__ float cv[kArgThreads * kTopK];
  __shared__ int ci[kArgThreads * kTopK];
  __shared__ int cand[kTopK];
  __shared__ double red[32];
  const int b = blockIdx.x;
  if (A.req_head && A.req_head[b] != A.head) return;  // another head serves this request
  const float* lg = A.logits + static_cast<long long>(b) * A.ld;
  // per-thread top-k (sorted descending; ties keep the lower index first)
  float v[kTopK];
  int ix[kTopK];
#pragma unroll
  for (int k = 0; k < kTopK; ++k) {
    v[k] = -INFINITY;
    ix[k] = 0x7fffffff;
  }
  // merge the sorted per-thread lists in registers: each round the warp's best head (value,
  // then lower index) is taken and its owner lane shifts its list; warps' top-k go to shared
  // memory and warp 0 merges those the same way
  auto warp_topk = [&](float* hv, int* hi, float* out_v, int* out_i) {
    const int lane = threadIdx.x & 31;
    for (int k = 0; k < kTopK; ++k) {
      float bv = hv[0];
      int bi = hi[0];
      int bl = lane;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        const int ol = __shfl_xor_sync(0xffffffffu, bl, o);
        if (ov > bv || (ov == bv && oi < bi)) {
          bv = ov;
          bi = oi;
          bl = ol;
        }
      }
      if (lane == bl) {  // the winner drops its head
#pragma unroll
        for (int t = 0; t < kTopK - 1; ++t) {
          hv[t] = hv[t + 1];
          hi[t] = hi[t + 1];
        }
        hv[kTopK - 1] = -INFINITY;
        hi[kTopK - 1] = 0x7fffffff;
      }
      if (lane == 0) {
        out_v[k] = bv;
        out_i[k] = bi;
      }
    }
  };
  // Two passes over the row. Pass 1: each thread's maximum (one FMNMX per logit); the block's
  // 8th-largest thread maximum tau is a lower bound of the row's 8th-largest logit (8 distinct
  // logits >= tau exist), so no logit < tau can be a candidate. Pass 2 (the row is L2-resident
  // from pass 1) offers only logits >= tau to the per-thread top-k, which keeps the insertion
  // -- ~40 predicated instructions per logit when offered every one -- off the common path.
  // The candidate set is the one an unfiltered scan selects (value, then lower index).
  constexpr int kRound = 8;  // 32 logits in flight per thread: 8 x float4 per round
  const int V4 = A.V & ~3;   // rows are 16-byte aligned (ld % 4 == 0)
  __shared__ float tau_s;
  {
    float tmax = -INFINITY;
    int j0 = threadIdx.x * 4;
    for (; j0 + (kRound - 1) * 4 * kArgThreads < V4; j0 += kRound * 4 * kArgThreads) {
      float4 x4[kRound];
#pragma unroll
      for (int t = 0; t < kRound; ++t)
        x4[t] = *reinterpret_cast<const float4*>(lg + j0 + t * 4 * kArgThreads);
#pragma unroll
      for (int t = 0; t < kRound; ++t)
        tmax = fmaxf(tmax, fmaxf(fmaxf(x4[t].x, x4[t].y), fmaxf(x4[t].z, x4[t].w)));
    }
    for (; j0 < V4; j0 += 4 * kArgThreads) {
      const float4 x4 = *reinterpret_cast<const float4*>(lg + j0);
      tmax = fmaxf(tmax, fmaxf(fmaxf(x4.x, x4.y), fmaxf(x4.z, x4.w)));
    }
    for (int j = V4 + static_cast<int>(threadIdx.x); j < A.V; j += kArgThreads) tmax = fmaxf(tmax, lg[j]);
    float hv[kTopK];
    int hi[kTopK];
#pragma unroll
    for (int k = 0; k < kTopK; ++k) {
      hv[k] = k == 0 ? tmax : -INFINITY;
      hi[k] = k == 0 ? static_cast<int>(threadIdx.x) : 0x7fffffff;
    }
    warp_topk(hv, hi, cv + (threadIdx.x >> 5) * kTopK, ci + (threadIdx.x >> 5) * kTopK);
    __syncthreads();
    if (threadIdx.x < 32) {
#pragma unroll
      for (int t = 0; t < kTopK; ++t) {
        const bool own = static_cast<int>(threadIdx.x) < kArgThreads / 32;
        hv[t] = own ? cv[threadIdx.x * kTopK + t] : -INFINITY;
        hi[t] = own ? ci[threadIdx.x * kTopK + t] : 0x7fffffff;
      }
      float tv[kTopK];
      int ti[kTopK];
      warp_topk(hv, hi, tv, ti);
      if (threadIdx.x == 0) tau_s = tv[kTopK - 1];
    }
    __syncthreads();
  }
  const float tau = tau_s;
  auto consider = [&](float x, int xi) {
    if (x > v[kTopK - 1]) {  // insert, keeping the earlier index first among equals
#pragma unroll
      for (int k = 0; k < kTopK; ++k) {
        if (x > v[k]) {
          const float tv = v[k];
          const int ti = ix[k];
          v[k] = x;
          ix[k] = xi;
          x = tv;
          xi = ti;
        }
      }
    }
  };
  auto consider4 = [&](const float4& x4, int jj) {
    if (fmaxf(fmaxf(x4.x, x4.y), fmaxf(x4.z, x4.w)) >= tau) {
      consider(x4.x, jj);
      consider(x4.y, jj + 1);
      consider(x4.z, jj + 2);
      consider(x4.w, jj + 3);
    }
  };
  int j0 = threadIdx.x * 4;
  for (; j0 + (kRound - 1) * 4 * kArgThreads < V4; j0 += kRound * 4 * kArgThreads) {
    float4 x4[kRound];
#pragma unroll
    for (int t = 0; t < kRound; ++t)
      x4[t] = __ldcs(reinterpret_cast<const float4*>(lg + j0 + t * 4 * kArgThreads));
#pragma unroll
    for (int t = 0; t < kRound; ++t) consider4(x4[t], j0 + t * 4 * kArgThreads);
  }
  for (; j0 < V4; j0 += 4 * kArgThreads) consider4(*reinterpret_cast<const float4*>(lg + j0), j0);
  for (int j = V4 + static_cast<int>(threadIdx.x); j < A.V; j += kArgThreads) {
    if (lg[j] >= tau) consider(lg[j], j);
  }
  warp_topk(v, ix, cv + (threadIdx.x >> 5) * kTopK, ci + (threadIdx.x >> 5) * kTopK);
  __syncthreads();
  if (threadIdx.x < 32) {
    // kArgThreads / 32 warps x kTopK candidates: lane l takes warp l's list when l < #warps
    float hv[kTopK];
    int hi[kTopK];
#pragma unroll
    for (int t = 0; t < kTopK; ++t) {
      const bool own = static_cast<int>(threadIdx.x) < kArgThreads / 32;
      hv[t] = own ? cv[threadIdx.x * kTopK + t] : -INFINITY;
      hi[t] = own ? ci[threadIdx.x * kTopK + t] : 0x7fffffff;
    }
    float tv[kTopK];
    int ti[kTopK];
    warp_topk(hv, hi, tv, ti);
    if (threadIdx.x == 0) {
#pragma unroll
      for (int k = 0; k < kTopK; ++k) cand[k] = ti[k] < A.V ? ti[k] : -1;
    }
  }
  __syncthreads();
  // f64 rescoring of the candidates: h (f32 row) . W[:, j] + b[j] (project_row, model.cpp:130-136),
  // all candidates in one pass over the row (independent loads), one block reduction
  const float* h = A.h32 + static_cast<long long>(b) * A.d;
  int cj[kTopK];
#pragma unroll
  for (int k = 0; k < kTopK; ++k) cj[k] = cand[k];
  double acc[kTopK];
#pragma unroll
  for (int k = 0; k < kTopK; ++k) acc[k] = 0.0;
  if (A.wT) {  // same order of sums per thread; the weights read from contiguous rows
    for (int i = threadIdx.x; i < A.d; i += blockDim.x) {
      const double hv = static_cast<double>(h[i]);
#pragma unroll
      for (int k = 0; k < kTopK; ++k) {
        if (cj[k] >= 0) acc[k] += hv * static_cast<double>(__ldg(A.wT + static_cast<long long>(cj[k]) * A.d + i));
      }
    }
  } else {
    for (int i = threadIdx.x; i < A.d; i += blockDim.x) {
      const double hv = static_cast<double>(h[i]);
      const float* wr = A.w + static_cast<long long>(i) * A.V;
#pragma unroll
      for (int k = 0; k < kTopK; ++k) {
        if (cj[k] >= 0) acc[k] += hv * static_cast<double>(__ldg(wr + cj[k]));
      }
    }
  }
  __shared__ double red8[kTopK][kArgThreads / 32];
  const int wid = threadIdx.x >> 5, lid = threadIdx.x & 31;
#pragma unroll
  for (int k = 0; k < kTopK; ++k) {
    double t = acc[k];
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (lid == 0) red8[k][wid] = t;
  }
  __syncthreads();
  double best = -INFINITY;
  int besti = 0x7fffffff;
#pragma unroll
  for (int k = 0; k < kTopK; ++k) {
    const int j = cj[k];
    if (j < 0) continue;
    double t = 0.0;
    for (int w = 0; w < kArgThreads / 32; ++w) t += red8[k][w];
    t += static_cast<double>(A.bias[j]);
    if (t > best || (t == best && j < besti)) {
      best = t;
      besti = j;
    }
  }
  if (threadIdx.x == 0) {
    const int tok = besti == 0x7fffffff ? 0 : besti;
    if (A.labels_out) A.labels_out[b] = tok;
    if (A.scores_out) A.scores_out[static_cast<long long>(b) * A.scores_ld] = static_cast<float>(best);
    if (A.gen_tokens) {
      int pos = A.gen_pos[b];
      if (A.advance) A.gen_pos[b] = ++pos;
      A.gen_tokens[static_cast<long long>(b) * A.tok_stride + pos] = static_cast<uint32_t>(tok);
      const int st = A.step >= 0 ? A.step : pos - A.lens[b];
      A.out_tokens[static_cast<long long>(b) * A.out_ld + st] = tok;
      if (A.out_logits) A.out_logits[static_cast<long long>(b) * A.out_ld + st] = static_cast<float>(best);
    }
  }
}

// ---------------------------------------------------------------------------
// One CTA per (head, request): q of the new row against keys 0..pos.
__global__ void __launch_bounds__(128) attn_decode_kernel(AttnDecodeArgs A) {
  extern __shared__ float sc[];  // [pos + 1] scores, then 4 x 64 partial contexts
  __shared__ float qs[64];
  __shared__ float red[32];
  const int h = blockIdx.x, b = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int d = A.d;
  const int pos = A.gen_pos[b];
  const int len0 = A.lens[b];
  const int nk = pos + 1;
  const uint16_t* qrow = A.qkv_new + static_cast<long long>(b) * 3 * d;
  if (threadIdx.x < 64) qs[threadIdx.x] = ld16(qrow, h * 64 + threadIdx.x, A.bf16);
  // append this row's k, v (head slice) to the generated-rows cache
  uint16_t* trow = A.tail + (static_cast<long long>(b) * A.tail_cap + (pos - len0)) * 2 * d;
  if (threadIdx.x < 64) {
    const uint32_t* src = reinterpret_cast<const uint32_t*>(qrow + d + h * 64);
    uint32_t* dst = reinterpret_cast<uint32_t*>(trow + h * 64);
    if (threadIdx.x < 32) dst[threadIdx.x] = src[threadIdx.x];
    else {
      reinterpret_cast<uint32_t*>(trow + d + h * 64)[threadIdx.x - 32] =
          reinterpret_cast<const uint32_t*>(qrow + 2 * d + h * 64)[threadIdx.x - 32];
    }
  }
  // key / value rows without branches (selects), so unrolled loads issue back to back:
  // prefill rows j < len0, generated rows len0 <= j < pos, the new row j == pos
  const uint16_t* pre = A.qkv_prefill + static_cast<long long>(b) * A.S * 3 * d + d + h * 64;
  const uint16_t* gen = A.tail + static_cast<long long>(b) * A.tail_cap * 2 * d + h * 64 -
                        static_cast<long long>(len0) * 2 * d;
  const uint16_t* cur = qrow + d + h * 64;
  auto key_ptr = [&](int j) -> const uint16_t* {
    const uint16_t* p = j < len0 ? pre + static_cast<long long>(j) * 3 * d
                                 : gen + static_cast<long long>(j) * 2 * d;
    return j == pos ? cur : p;
  };
  auto val_ptr = [&](int j) -> const uint16_t* { return key_ptr(j) + d; };
  __syncthreads();
  // scores: one key per thread (its 64-dim head slice as 8 x 16-byte loads), no shuffles
  for (int j = threadIdx.x; j < nk; j += blockDim.x) {
    const uint4* kp = reinterpret_cast<const uint4*>(key_ptr(j));
    uint4 u[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) u[c] = kp[c];
    float s = 0.f;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      float f[8];
      unpack8(u[c], f, A.bf16);
#pragma unroll
      for (int i = 0; i < 8; ++i) s += f[i] * qs[8 * c + i];
    }
    sc[j] = s * A.scale;
  }
  __syncthreads();
  float m = -INFINITY;
  for (int j = threadIdx.x; j < nk; j += blockDim.x) m = fmaxf(m, sc[j]);
  m = block_max_f(m, red);
  float sum = 0.f;
  for (int j = threadIdx.x; j < nk; j += blockDim.x) {
    const float e = __expf(sc[j] - m);
    sc[j] = e;
    sum += e;
  }
  sum = block_sum_t(sum, red);  // contains the barrier that publishes sc[]
  // context: warp w takes keys j = w (mod 4), lane its two dims; 8 keys in flight per warp
  float a0 = 0.f, a1 = 0.f;
  int j = warp;
  for (; j + 28 < nk; j += 32) {
    uint32_t u[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) u[t] = reinterpret_cast<const uint32_t*>(val_ptr(j + 4 * t))[lane];
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const float2 v = A.bf16 ? make_float2(__uint_as_float(u[t] << 16), __uint_as_float(u[t] & 0xffff0000u))
                              : __half22float2(*reinterpret_cast<const __half2*>(&u[t]));
      const float p = sc[j + 4 * t];
      a0 += p * v.x;
      a1 += p * v.y;
    }
  }
  for (; j < nk; j += 4) {
    const uint32_t u = reinterpret_cast<const uint32_t*>(val_ptr(j))[lane];
    const float2 v = A.bf16 ? make_float2(__uint_as_float(u << 16), __uint_as_float(u & 0xffff0000u))
                            : __half22float2(*reinterpret_cast<const __half2*>(&u));
    const float p = sc[j];
    a0 += p * v.x;
    a1 += p * v.y;
  }
  float* part = sc + ((nk + 3) & ~3);
  part[warp * 64 + 2 * lane] = a0;
  part[warp * 64 + 2 * lane + 1] = a1;
  __syncthreads();
  if (threadIdx.x < 64) {
    const int c = threadIdx.x;
    const float o = (part[c] + part[64 + c] + part[128 + c] + part[192 + c]) / sum;
    A.ctx[static_cast<long long>(b) * d + h * 64 + c] = st16(o, A.bf16);
  }
}

// TMA-staged decode attention: one CTA per (head, request). Shared memory: the prompt's K and V
// head slices (S rows x 128 B each, SWIZZLE_128B: 16-byte chunk c of row r at (c ^ r % 8)) and
// the generated rows' K and V (tail_cap rows each); keys / values are read from shared memory
// only, the new row (j == pos) from this step's projections.
constexpr int kDecS = 256;     // max prompt rows staged (2 boxes of 128)
constexpr int kDecTailBox = 8; // generated rows per tail box (one 1 KB swizzle atom)
__global__ void __launch_bounds__(128) attn_decode_tma_kernel(const __grid_constant__ AttnDecodeMaps M,
                                                             AttnDecodeArgs A) {
  // the next decode GEMM (programmatic launch) may take free SM space during this grid's last
  // wave and stream its weights before its griddepcontrol.wait
  pdl_trigger();
  extern __shared__ uint8_t dsm[];
  uint8_t* base = dsm + ((1024 - (smem_u32(dsm) & 1023)) & 1023);
  const int S = A.S, T = A.tail_cap;
  uint8_t* kpre = base;                         // [S][128 B]
  uint8_t* vpre = kpre + S * 128;
  uint8_t* ktail = vpre + S * 128;              // [T][128 B] (1024-aligned: S % 128 == 0)
  uint8_t* vtail = ktail + ((T * 128 + 1023) & ~1023);
  float* sc = reinterpret_cast<float*>(vtail + ((T * 128 + 1023) & ~1023));  // [S + T] scores
  __shared__ float qs[64];
  __shared__ float red[32];
  __shared__ __align__(16) float part[4 * 64];
  __shared__ uint64_t bar_k, bar_v;  // K lands first: scores and softmax overlap the V copy
  const int h = blockIdx.x, b = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int d = A.d;
  const int pos = A.gen_pos[b];
  const int len0 = A.lens[b];
  const int nk = pos + 1;
  const int n_tail = pos - len0;  // generated rows already cached
  const uint16_t* qrow = A.qkv_new + static_cast<long long>(b) * 3 * d;
  if (threadIdx.x == 0) {
    mbar_init(&bar_k, 1);
    mbar_init(&bar_v, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const int nbox = (len0 + 127) / 128;
    const int ntail = (n_tail + kDecTailBox - 1) / kDecTailBox;  // only the cached rows
    const uint32_t bytes = nbox * 16384 + ntail * kDecTailBox * 128;
    mbar_arrive_expect_tx(&bar_k, bytes);
    mbar_arrive_expect_tx(&bar_v, bytes);
    for (int x = 0; x < nbox; ++x)
      tma_load_2d(kpre + x * 16384, &M.prefill, &bar_k, d + h * 64, b * S + 128 * x);
    for (int x = 0; x < ntail; ++x)
      tma_load_2d(ktail + x * kDecTailBox * 128, &M.tail, &bar_k, h * 64, b * T + kDecTailBox * x);
    for (int x = 0; x < nbox; ++x)
      tma_load_2d(vpre + x * 16384, &M.prefill, &bar_v, 2 * d + h * 64, b * S + 128 * x);
    for (int x = 0; x < ntail; ++x)
      tma_load_2d(vtail + x * kDecTailBox * 128, &M.tail, &bar_v, d + h * 64, b * T + kDecTailBox * x);
  }
  // launched as a programmatic dependent of the QKV GEMM: everything above reads only the prompt
  // and earlier steps' cache rows; this step's q, k, v are read from here on
  pdl_wait();
  if (threadIdx.x < 64) qs[threadIdx.x] = ld16(qrow, h * 64 + threadIdx.x, A.bf16);
  __syncthreads();
  // append this row's k, v (head slice) to the generated-rows cache (global; the staged copy of
  // that row is never read: j == pos comes from qkv_new)
  if (threadIdx.x < 64) {
    uint16_t* trow = A.tail + (static_cast<long long>(b) * T + n_tail) * 2 * d;
    if (threadIdx.x < 32) {
      reinterpret_cast<uint32_t*>(trow + h * 64)[threadIdx.x] =
          reinterpret_cast<const uint32_t*>(qrow + d + h * 64)[threadIdx.x];
    } else {
      reinterpret_cast<uint32_t*>(trow + d + h * 64)[threadIdx.x - 32] =
          reinterpret_cast<const uint32_t*>(qrow + 2 * d + h * 64)[threadIdx.x - 32];
    }
  }
  mbar_wait(&bar_k, 0);
  // row r of a staged operand: 8 chunks of 16 B, swizzled
  auto srow = [&](const uint8_t* box, int r, int c) -> const uint4* {
    return reinterpret_cast<const uint4*>(box + r * 128 + ((c ^ (r & 7)) << 4));
  };
  for (int j = threadIdx.x; j < nk; j += blockDim.x) {
    float s = 0.f;
    if (j == pos) {
      const uint4* kp = reinterpret_cast<const uint4*>(qrow + d + h * 64);
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        float f[8];
        unpack8(kp[c], f, A.bf16);
#pragma unroll
        for (int i = 0; i < 8; ++i) s += f[i] * qs[8 * c + i];
      }
    } else {
      const uint8_t* box = j < len0 ? kpre : ktail;
      const int r = j < len0 ? j : j - len0;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        float f[8];
        unpack8(*srow(box, r, c), f, A.bf16);
#pragma unroll
        for (int i = 0; i < 8; ++i) s += f[i] * qs[8 * c + i];
      }
    }
    sc[j] = s * A.scale;
  }
  __syncthreads();
  float m = -INFINITY;
  for (int j = threadIdx.x; j < nk; j += blockDim.x) m = fmaxf(m, sc[j]);
  m = block_max_f(m, red);
  float sum = 0.f;
  for (int j = threadIdx.x; j < nk; j += blockDim.x) {
    const float e = __expf(sc[j] - m);
    sc[j] = e;
    sum += e;
  }
  sum = block_sum_t(sum, red);  // contains the barrier that publishes sc[]
  mbar_wait(&bar_v, 0);
  // context: 8 lanes per value row, lane c its 16-byte chunk c (dims 8c..8c+7); the CTA's 16 lane
  // groups take rows g, g + 16, ... of the prompt box, then of the generated rows' box, then
  // group 15 the new row from this step's projections
  const int g = threadIdx.x >> 3, c = lane & 7;
  float acc[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) acc[e] = 0.f;
  auto fma_row = [&](const uint4& u, float p) {
    float f[8];
    unpack8(u, f, A.bf16);
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] += p * f[e];
  };
  for (int r = g; r < len0; r += 16) fma_row(*srow(vpre, r, c), sc[r]);
  for (int r = g; r < n_tail; r += 16) fma_row(*srow(vtail, r, c), sc[len0 + r]);
  if (g == 15) fma_row(reinterpret_cast<const uint4*>(qrow + 2 * d + h * 64)[c], sc[pos]);
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    acc[e] += __shfl_xor_sync(0xffffffffu, acc[e], 8);
    acc[e] += __shfl_xor_sync(0xffffffffu, acc[e], 16);
  }
  if (lane < 8) {
    float4* pw = reinterpret_cast<float4*>(part + warp * 64 + c * 8);
    pw[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
    pw[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
  }
  __syncthreads();
  if (threadIdx.x < 64) {
    const int cc = threadIdx.x;
    const float o = (part[cc] + part[64 + cc] + part[128 + cc] + part[192 + cc]) / sum;
    A.ctx[static_cast<long long>(b) * d + h * 64 + cc] = st16(o, A.bf16);
  }
}

// ---------------------------------------------------------------------------
// One CTA per decode row: y = relu(ctx.Wc + bc).Wu + bu + a + h, x = LN1(y), where the slot's
// folded down projection Wc = Wo.Wd, bc = bo.Wd + bd (adapter.cu) makes relu(ctx.Wc + bc) the
// reference's relu(a.Wd + bd).
// RP > 0: bottleneck fixed at compile time (all weight loads of a unit / an output in flight)
template <int RP>
__global__ void __launch_bounds__(256) adapter_rows_ln_kernel(AdapterRowsArgs A) {
  pdl_trigger();  // as in attn_decode_tma_kernel: FFN1 may start streaming its weights
  extern __shared__ float sm[];  // ctx[d] (the down projection's input), y[d], mid[r_pad]
  __shared__ float red[32];
  const int b = blockIdx.x;
  const int d = A.d, rp = RP > 0 ? RP : A.r_pad;
  float* a = sm;
  float* y = sm + d;
  float* mid = sm + 2 * d;
  const int task = A.req_task[b];
  int slot = task >= 0 ? A.slot_of[static_cast<long long>(task) * A.layers + A.layer] : -1;
  if (slot < 0) {
    if (threadIdx.x == 0) atomicExch(A.err, HMI_SCHEDULING_BUG);
    slot = 0;
  }
  const uint8_t* base = A.arena + static_cast<size_t>(slot) * A.slot_bytes;
  const uint16_t* wd = reinterpret_cast<const uint16_t*>(base);          // [r_pad][d]
  const uint16_t* wu = wd + static_cast<size_t>(rp) * d;                 // [d][r_pad]
  const float* bd = reinterpret_cast<const float*>(wu + static_cast<size_t>(d) * rp);
  const float* bu = bd + rp;
  const uint16_t* arow = A.ctx16 + static_cast<long long>(b) * d;
  const uint16_t* skiprow = A.a16 + static_cast<long long>(b) * d;  // the adapter's skip input
  const uint16_t* hrow = A.h16 + static_cast<long long>(b) * d;
  // down projection (fast form): warp per bottleneck unit, 16-byte weight vectors across the
  // lanes; every weight load of this warp's 8 units in flight at once. The tenant slot is
  // resident for the whole generate call, so these loads go out before griddepcontrol.wait
  // (this kernel is a programmatic dependent of the O projection, which triggers at entry)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  constexpr int U = RP > 0 ? RP / 8 : 1;
  const bool fast_down = RP == 64 && nw == 8 && d <= 96 * 8;
  const int nch = d / 8;
  uint4 w[U][3];
  float bdl = 0.f;
  if (fast_down) {
    bdl = lane < U ? bd[warp + 8 * lane] : 0.f;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint4* w4 = reinterpret_cast<const uint4*>(wd + static_cast<size_t>(warp + 8 * u) * d);
#pragma unroll
      for (int m = 0; m < 3; ++m) {
        const int c = lane + 32 * m;
        w[u][m] = c < nch ? __ldg(w4 + c) : make_uint4(0, 0, 0, 0);
      }
    }
  }
  pdl_wait();  // ctx (attention), a (O projection), h (LayerNorm) from here on
  for (int c = threadIdx.x; c < d / 8; c += blockDim.x) {
    float f[8];
    unpack8(reinterpret_cast<const uint4*>(arow)[c], f, A.bf16);
#pragma unroll
    for (int e = 0; e < 8; ++e) a[c * 8 + e] = f[e];
  }
  // the up phase's per-output inputs (bias, skip, residual), in flight with the down phase
  // coalesced up phase (below): lane group g = tid / 8 reads rows g + 32 k of the up projection,
  // lane c = tid % 8 chunk c of each, and owns the outputs of rows k = c, c + 8, c + 16
  const bool fast_up = RP == 64 && blockDim.x == 256 && d % 256 == 0 && d <= 768;
  const int ug = threadIdx.x >> 3, uc = threadIdx.x & 7;
  float ub[3] = {0.f, 0.f, 0.f}, us[3] = {0.f, 0.f, 0.f}, uh[3] = {0.f, 0.f, 0.f};
  if (fast_up) {
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const int i = ug + 32 * (uc + 8 * k);
      if (i < d) {
        ub[k] = bu[i];
        us[k] = ld16(skiprow, i, A.bf16);
        uh[k] = ld16(hrow, i, A.bf16);
      }
    }
  }
  __syncthreads();
  if (fast_down) {
    // same per-lane order of sums as the general loop below, so the same mid[]
#pragma unroll
    for (int u = 0; u < U; ++u) {
      float acc = 0.f;
#pragma unroll
      for (int m = 0; m < 3; ++m) {
        const int c = lane + 32 * m;
        if (c < nch) {
          float f[8];
          unpack8(w[u][m], f, A.bf16);
#pragma unroll
          for (int e = 0; e < 8; ++e) acc += a[c * 8 + e] * f[e];
        }
      }
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      const float bias = __shfl_sync(0xffffffffu, bdl, u);
      if (lane == 0) mid[warp + 8 * u] = fmaxf(acc + bias, 0.f);
    }
  } else {
    for (int j = warp; j < rp; j += nw) {
      const uint4* w4 = reinterpret_cast<const uint4*>(wd + static_cast<size_t>(j) * d);
      float acc = 0.f;
      for (int c = lane; c < d / 8; c += 32) {
        float f[8];
        unpack8(__ldg(w4 + c), f, A.bf16);
#pragma unroll
        for (int e = 0; e < 8; ++e) acc += a[c * 8 + e] * f[e];
      }
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane == 0) mid[j] = fmaxf(acc + bd[j], 0.f);
    }
  }
  __syncthreads();
  // the GEMM path rounds the bottleneck activations to 16 bits; so does this one
  for (int j = threadIdx.x; j < rp; j += blockDim.x) {
    const uint16_t u = st16(mid[j], A.bf16);
    mid[j] = A.bf16 ? __uint_as_float(static_cast<uint32_t>(u) << 16) : __half2float(__ushort_as_half(u));
  }
  __syncthreads();
  // up projection + bias + skip + residual
  float s1 = 0.f;
  if (fast_up) {
    // each warp instruction reads four consecutive 128-byte rows (512 contiguous bytes); every
    // weight load of the group's d / 32 rows in flight at once; row sums reduced over the 8 lanes
    constexpr int KR = 24;
    const int nr = d / 32;
    const uint4* w4 = reinterpret_cast<const uint4*>(wu);
    uint4 w[KR];
#pragma unroll
    for (int k = 0; k < KR; ++k)
      w[k] = k < nr ? __ldg(w4 + static_cast<size_t>(ug + 32 * k) * 8 + uc) : make_uint4(0, 0, 0, 0);
    float m8[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) m8[e] = mid[uc * 8 + e];
    float mine[3] = {0.f, 0.f, 0.f};
#pragma unroll
    for (int k = 0; k < KR; ++k) {
      if (k >= nr) break;
      float f[8];
      unpack8(w[k], f, A.bf16);
      float p = 0.f;
#pragma unroll
      for (int e = 0; e < 8; ++e) p += m8[e] * f[e];
      p += __shfl_xor_sync(0xffffffffu, p, 1);
      p += __shfl_xor_sync(0xffffffffu, p, 2);
      p += __shfl_xor_sync(0xffffffffu, p, 4);
      if ((k & 7) == uc) mine[k >> 3] = p;
    }
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const int i = ug + 32 * (uc + 8 * j);
      if (uc + 8 * j < nr) {
        const float v = mine[j] + ub[j] + us[j] + uh[j];
        y[i] = v;
        s1 += v;
      }
    }
  } else
  for (int i = threadIdx.x; i < d; i += blockDim.x) {
    const uint4* w4 = reinterpret_cast<const uint4*>(wu + static_cast<size_t>(i) * rp);
    float acc = 0.f;
    if constexpr (RP > 0) {
      uint4 w[RP / 8];
#pragma unroll
      for (int c = 0; c < RP / 8; ++c) w[c] = __ldg(w4 + c);
#pragma unroll
      for (int c = 0; c < RP / 8; ++c) {
        float f[8];
        unpack8(w[c], f, A.bf16);
#pragma unroll
        for (int e = 0; e < 8; ++e) acc += mid[c * 8 + e] * f[e];
      }
    } else {
      for (int c = 0; c < rp / 8; ++c) {
        float f[8];
        unpack8(__ldg(w4 + c), f, A.bf16);
#pragma unroll
        for (int e = 0; e < 8; ++e) acc += mid[c * 8 + e] * f[e];
      }
    }
    const float v = acc + bu[i] + ld16(skiprow, i, A.bf16) + ld16(hrow, i, A.bf16);
    y[i] = v;
    s1 += v;
  }
  const float mean = block_sum_t(s1, red) / d;
  float s2 = 0.f;
  for (int i = threadIdx.x; i < d; i += blockDim.x) {
    const float t = y[i] - mean;
    s2 += t * t;
  }
  const float inv = 1.0f / sqrtf(block_sum_t(s2, red) / d + 1e-5f);
  for (int i = threadIdx.x; i < d; i += blockDim.x)
    A.x16[static_cast<long long>(b) * d + i] = st16((y[i] - mean) * inv * A.ln_g[i] + A.ln_b[i], A.bf16);
}

}  // namespace

void launch_lm_gather(const void* y16, const float* h32, const float* gamma, const float* beta,
                      const int* lens, int n_req, int S, int d, int precision, float* out32,
                      void* out16, cudaStream_t stream) {
  if (n_req <= 0) return;
  const size_t smem = static_cast<size_t>(d) * sizeof(double);
  lm_gather_kernel<<<n_req, 256, smem, stream>>>(static_cast<const uint16_t*>(y16), h32, gamma,
                                                 beta, lens, S, d, precision, out32,
                                                 static_cast<uint16_t*>(out16));
  HMI_CUDA(cudaGetLastError());
}

void launch_lm_argmax(const LmArgmaxArgs& a, int n_req, cudaStream_t stream) {
  if (n_req <= 0) return;
  lm_argmax_kernel<<<n_req, kArgThreads, 0, stream>>>(a);
  HMI_CUDA(cudaGetLastError());
}

void launch_attn_decode(const AttnDecodeArgs& a, int n_req, int heads, int max_keys,
                        cudaStream_t stream) {
  if (n_req <= 0) return;
  const size_t smem = (static_cast<size_t>((max_keys + 3) & ~3) + 4 * 64) * sizeof(float);
  if (smem > 48 * 1024) {
    HMI_CUDA(cudaFuncSetAttribute(attn_decode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
  }
  attn_decode_kernel<<<dim3(heads, n_req), 128, smem, stream>>>(a);
  HMI_CUDA(cudaGetLastError());
}

bool attn_decode_tma_ok(int S, int tail_cap) {
  return S % 128 == 0 && S <= kDecS && tail_cap >= 1 && tail_cap <= 256;
}

AttnDecodeMaps make_attn_decode_maps(const void* qkv_prefill, int max_rows, void* tail,
                                     int max_batch, int tail_cap, int d, int precision) {
  const CUtensorMapDataType t16 =
      precision == 1 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  AttnDecodeMaps m;
  m.prefill = make_tmap_2d(qkv_prefill, t16, 3ull * d, max_rows, 3ull * d * 2, 64, 128,
                           CU_TENSOR_MAP_SWIZZLE_128B);
  m.tail = make_tmap_2d(tail, t16, 2ull * d, static_cast<uint64_t>(max_batch) * tail_cap,
                        2ull * d * 2, 64, kDecTailBox, CU_TENSOR_MAP_SWIZZLE_128B);
  return m;
}

void launch_attn_decode_tma(const AttnDecodeArgs& a, const AttnDecodeMaps& m, int n_req,
                            int heads, cudaStream_t stream) {
  if (n_req <= 0) return;
  HMI_CHECK(attn_decode_tma_ok(a.S, a.tail_cap) && a.d == heads * 64, HMI_CONFIG_ERROR,
            "decode attention: staged form needs S % 128 == 0, S <= 256, tail <= 256, dh 64");
  const size_t tail_b = (static_cast<size_t>(a.tail_cap) * 128 + 1023) & ~static_cast<size_t>(1023);
  const size_t smem = 1024 + 2 * static_cast<size_t>(a.S) * 128 + 2 * tail_b +
                      static_cast<size_t>(a.S + a.tail_cap + 4) * 4;
  static size_t configured = 0;
  if (smem > configured) {
    HMI_CUDA(cudaFuncSetAttribute(attn_decode_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
    configured = smem;
  }
  // programmatic dependent of the QKV GEMM (which triggers at entry): the cached K / V copies are
  // issued before griddepcontrol.wait, under the GEMM
  launch_pdl(attn_decode_tma_kernel, dim3(heads, n_req), dim3(128), smem, stream, m, a);
}

void launch_adapter_rows_ln(const AdapterRowsArgs& a, int n_req, cudaStream_t stream) {
  if (n_req <= 0) return;
  HMI_CHECK(a.d % 8 == 0 && a.r_pad % 8 == 0, HMI_CONFIG_ERROR, "adapter rows: d, r_pad % 8");
  const size_t smem = static_cast<size_t>(2 * a.d + a.r_pad) * sizeof(float);
  if (a.r_pad == 64) {
    launch_pdl(adapter_rows_ln_kernel<64>, dim3(n_req), dim3(256), smem, stream, a);
  } else {
    launch_pdl(adapter_rows_ln_kernel<0>, dim3(n_req), dim3(256), smem, stream, a);
  }
  HMI_CUDA(cudaGetLastError());
}

}  // namespace hmi_b200
