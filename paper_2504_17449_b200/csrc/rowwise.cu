// SPDX-License-Identifier: Apache-2.0
//
// HBM-bound row-wise kernels of the hot path:
//   K4 LayerNorm            layer_norm (proj/src/tensor/ops.cpp:92-116)
//   K5 PLOT retrieval       retrieve_sequence / resolve_window / VersionTree::lookup
//                           (proj/src/plot/retrieval.cpp:23-124, version_tree.cpp:47-79)
//   K6 routing              InstanceTable (scheduler/request.hpp:30-36) + slot mapping
//   K7 task head            apply_head / argmax (proj/src/transformer/model.cpp:120-171)
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "kernels.hpp"

namespace hmi_b200 {

namespace {

template <bool kBf16>
__device__ __forceinline__ float2 unpack16x2(uint32_t u) {
  if constexpr (kBf16) {
    return make_float2(__uint_as_float(u << 16), __uint_as_float(u & 0xffff0000u));
  } else {
    return __half22float2(*reinterpret_cast<const __half2*>(&u));
  }
}

template <bool kBf16>
__device__ __forceinline__ uint32_t pack16x2(float a, float b) {
  if constexpr (kBf16) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
  } else {
    __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
  }
}

// ---------------------------------------------------------------------------
// K4: one warp per row; d = 128 * V (V float4 per lane).
// ---------------------------------------------------------------------------
template <int V, bool kBf16>
__global__ void __launch_bounds__(256) layernorm_kernel(const float* __restrict__ y,
                                                        const float* __restrict__ gamma,
                                                        const float* __restrict__ beta,
                                                        uint16_t* __restrict__ out16,
                                                        float* __restrict__ out32, int rows,
                                                        int n_parts, long long part_stride,
                                                        const float* __restrict__ bias,
                                                        const uint16_t* __restrict__ res16) {
  constexpr int d = 128 * V;
  // a programmatically launched GEMM after this kernel may stream its weights during the
  // last wave (it still waits for this grid before reading the rows)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= rows) return;
  float4 v[V];
  if (n_parts == 0) {
    const float4* src = reinterpret_cast<const float4*>(y + static_cast<long long>(warp) * d);
#pragma unroll
    for (int i = 0; i < V; ++i) v[i] = __ldcs(src + lane + 32 * i);
  } else {
    // split-K partial sums (fixed order) + bias + 16-bit residual: the reduction of a split
    // GEMM folded into the LayerNorm that follows it
    const float4* bb = reinterpret_cast<const float4*>(bias);
    const uint2* rr = reinterpret_cast<const uint2*>(res16 + static_cast<long long>(warp) * d);
#pragma unroll
    for (int i = 0; i < V; ++i) v[i] = __ldcs(reinterpret_cast<const float4*>(y + static_cast<long long>(warp) * d) + lane + 32 * i);
    for (int sp = 1; sp < n_parts; ++sp) {
      const float4* src = reinterpret_cast<const float4*>(y + sp * part_stride + static_cast<long long>(warp) * d);
#pragma unroll
      for (int i = 0; i < V; ++i) {
        const float4 t = __ldcs(src + lane + 32 * i);
        v[i].x += t.x; v[i].y += t.y; v[i].z += t.z; v[i].w += t.w;
      }
    }
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const float4 b = __ldg(bb + lane + 32 * i);
      const uint2 u = rr[lane + 32 * i];
      const float2 r01 = unpack16x2<kBf16>(u.x), r23 = unpack16x2<kBf16>(u.y);
      v[i].x += b.x + r01.x; v[i].y += b.y + r01.y; v[i].z += b.z + r23.x; v[i].w += b.w + r23.y;
    }
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < V; ++i) s += (v[i].x + v[i].y) + (v[i].z + v[i].w);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  const float mean = s * (1.0f / d);
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < V; ++i) {
    const float a = v[i].x - mean, b = v[i].y - mean, c = v[i].z - mean, e = v[i].w - mean;
    q += (a * a + b * b) + (c * c + e * e);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
  const float inv = 1.0f / sqrtf(q * (1.0f / d) + 1e-5f);
  const float4* g4 = reinterpret_cast<const float4*>(gamma);
  const float4* b4 = reinterpret_cast<const float4*>(beta);
#pragma unroll
  for (int i = 0; i < V; ++i) {
    const int c4 = lane + 32 * i;
    const float4 g = __ldg(g4 + c4), b = __ldg(b4 + c4);
    float4 r;
    r.x = (v[i].x - mean) * inv * g.x + b.x;
    r.y = (v[i].y - mean) * inv * g.y + b.y;
    r.z = (v[i].z - mean) * inv * g.z + b.z;
    r.w = (v[i].w - mean) * inv * g.w + b.w;
    uint2 p;
    p.x = pack16x2<kBf16>(r.x, r.y);
    p.y = pack16x2<kBf16>(r.z, r.w);
    reinterpret_cast<uint2*>(out16 + static_cast<long long>(warp) * d)[c4] = p;
    if (out32) reinterpret_cast<float4*>(out32 + static_cast<long long>(warp) * d)[c4] = r;
  }
}

// ---------------------------------------------------------------------------
// K5: PLOT retrieval, one CTA per (request, 16-position chunk: 2.3 waves of 6 CTAs per SM instead of 1.15 at 32 — same-box 120 -> 108 us; 8 gives 116).
constexpr int kRetrieveChunk = 16;
// ---------------------------------------------------------------------------
__device__ __forceinline__ int32_t plot_find(const PlotDev& P, uint32_t version,
                                             const uint32_t* key, uint32_t len) {
  uint64_t i = plot_hash(version, len, key) & P.mask;
  for (;;) {
    const PlotSlot& s = P.slots[i];
    const uint32_t v = __ldg(&s.version);
    if (v == kEmptyKey) return -1;
    if (v == version && __ldg(&s.len) == len) {
      bool eq = true;
      for (uint32_t j = 0; j < len; ++j) eq &= (__ldg(&s.tok[j]) == key[j]);
      if (eq) return static_cast<int32_t>(__ldg(&s.row_base));
    }
    i = (i + 1) & P.mask;
  }
}

// VersionTree::lookup: the version's own table, then its parent chain to the root.
__device__ __forceinline__ int32_t plot_lookup(const PlotDev& P, int32_t version,
                                               const uint32_t* key, uint32_t len) {
  for (int depth = 0; version >= 0 && depth < 64; ++depth) {
    const int32_t r = plot_find(P, static_cast<uint32_t>(version), key, len);
    if (r >= 0) return r;
    version = __ldg(&P.parent[version]);
  }
  return -1;
}

// Phase 2 of K5 for one position: the mean of its cnt rep rows (ascending window order, f64,
// retrieval.cpp:114-122) for lane columns (lane + 32 i) * 4, i < V. GV float4 columns of every
// row are loaded before any is summed, so a warp keeps cnt * GV * 512 B in flight.
template <int V, int NG, int GV>
__device__ __forceinline__ void gather_mean(const float* __restrict__ reps, const int32_t* rows,
                                            int cnt, int d, int lane, long long orow, void* h16,
                                            int bf16, double* h64) {
  const double inv = cnt > 0 ? 1.0 / static_cast<double>(cnt) : 0.0;
  const float4* src[NG];
#pragma unroll
  for (int k = 0; k < NG; ++k)
    src[k] = reinterpret_cast<const float4*>(reps + static_cast<long long>(rows[k] < 0 ? 0 : rows[k]) * d) + lane;
#pragma unroll
  for (int g = 0; g < V; g += GV) {
    float4 xs[NG][GV];
#pragma unroll
    for (int k = 0; k < NG; ++k) {
      if (k < cnt) {
#pragma unroll
        for (int j = 0; j < GV; ++j)
          if (g + j < V) xs[k][j] = __ldg(src[k] + 32 * (g + j));
      }
    }
#pragma unroll
    for (int j = 0; j < GV; ++j) {
      if (g + j < V) {
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
        for (int k = 0; k < NG; ++k) {
          if (k < cnt) {
            a0 = a0 + static_cast<double>(xs[k][j].x);
            a1 = a1 + static_cast<double>(xs[k][j].y);
            a2 = a2 + static_cast<double>(xs[k][j].z);
            a3 = a3 + static_cast<double>(xs[k][j].w);
          }
        }
        a0 *= inv; a1 *= inv; a2 *= inv; a3 *= inv;
        const int col = (lane + 32 * (g + j)) * 4;
        if (h64) {
          double* o = h64 + orow * d + col;
          o[0] = a0; o[1] = a1; o[2] = a2; o[3] = a3;
        }
        const float f0 = __double2float_rn(a0), f1 = __double2float_rn(a1);
        const float f2 = __double2float_rn(a2), f3 = __double2float_rn(a3);
        uint2 pk;
        if (bf16) {
          pk.x = pack16x2<true>(f0, f1);
          pk.y = pack16x2<true>(f2, f3);
        } else {
          pk.x = pack16x2<false>(f0, f1);
          pk.y = pack16x2<false>(f2, f3);
        }
        *reinterpret_cast<uint2*>(static_cast<uint16_t*>(h16) + orow * d + col) = pk;
      }
    }
  }
}

template <int V, int NG, int GV, int MINB>
__global__ void __launch_bounds__(256, MINB) retrieve_kernel(PlotDev P, const uint32_t* __restrict__ tokens,
                                                       const int* __restrict__ lens,
                                                       const int* __restrict__ req_version,
                                                       int S, int causal, void* __restrict__ h16,
                                                       int bf16, double* __restrict__ h64,
                                                       int32_t* __restrict__ gather,
                                                       int32_t* __restrict__ levels,
                                                       int32_t* __restrict__ err,
                                                       const int32_t* __restrict__ dec_pos,
                                                       int tok_stride) {
  constexpr int kMaxWin = kRetrieveChunk + kMaxNgram;
  __shared__ int32_t wrow[kMaxWin * kMaxNgram];  // rep row per (window, offset)
  __shared__ int32_t wlev[kMaxWin * kMaxNgram];  // sub-gram length
  const int n = P.ngram;
  const int b = blockIdx.x;
  // decode mode (dec_pos != null): the single causal row dec_pos[b] of a sequence
  // extended by generated tokens; output row b
  const int p0 = dec_pos ? dec_pos[b] : blockIdx.y * kRetrieveChunk;
  const int p1 = dec_pos ? p0 + 1 : (p0 + kRetrieveChunk < S ? p0 + kRetrieveChunk : S);
  const int len = dec_pos ? p0 + 1 : lens[b];
  const int version = req_version[b];
  const uint32_t* tok = tokens + static_cast<long long>(b) * (dec_pos ? tok_stride : S);
  const int hl = (n - 1) / 2, hr = n - 1 - hl;
  // windows this chunk of positions needs (encoder: centred windows covering them;
  // causal: the window ending at each position)
  const int c0 = causal ? p0 : (p0 - hr > 0 ? p0 - hr : 0);
  const int c1 = causal ? (p1 < len ? p1 : len) - 1 : (p1 - 1 + hl < len - 1 ? p1 - 1 + hl : len - 1);

  // ---- phase 1a: every (window, sub-gram, tree depth) probe of this chunk in parallel.
  // The version chain (VersionTree::lookup walks branch -> parent -> ... -> root,
  // version_tree.cpp:64-77) is resolved once; probe (w, o, k, depth) looks the sub-gram
  // tokens[start_w + o, +k) up in the depth-th table of the chain only.
  constexpr int kMaxDepth = 8;
  const int n_sub = n * (n + 1) / 2;           // valid (o, k) sub-grams of a full window
  extern __shared__ int32_t probe[];           // [window][sub-gram][P.max_depth]
  __shared__ int32_t chain[kMaxDepth];
  __shared__ int8_t sub_o[kMaxNgram * (kMaxNgram + 1) / 2], sub_k[kMaxNgram * (kMaxNgram + 1) / 2];
  __shared__ int32_t n_chain;
  if (threadIdx.x == 0) {
    int v = version, dd = 0;
    while (v >= 0 && dd < P.max_depth) {
      chain[dd++] = v;
      v = __ldg(&P.parent[v]);
    }
    n_chain = dd;
    int si = 0;
    for (int k = 1; k <= n; ++k)
      for (int o = 0; o + k <= n; ++o) {
        sub_o[si] = static_cast<int8_t>(o);
        sub_k[si] = static_cast<int8_t>(k);
        ++si;
      }
  }
  __syncthreads();
  const int depth = n_chain;
  const int md = P.max_depth;
  const int n_win = c1 - c0 + 1;
  auto win_bounds = [&](int c, int& start, int& wl) {
    int end;
    if (causal) {
      start = c + 1 >= n ? c + 1 - n : 0;
      end = c;
    } else {
      start = c >= hl ? c - hl : 0;
      end = c + hr < len - 1 ? c + hr : len - 1;
    }
    wl = end - start + 1;
  };
  for (int t = threadIdx.x; t < n_win * n_sub * depth; t += blockDim.x) {
    const int dd = t % depth;
    const int si = (t / depth) % n_sub;
    const int wi = t / (depth * n_sub);
    const int o = sub_o[si], k = sub_k[si];
    int start, wl;
    win_bounds(c0 + wi, start, wl);
    int32_t r = -1;
    if (o + k <= wl) {
      uint32_t key[kMaxNgram];
      for (int j = 0; j < k; ++j) key[j] = tok[start + o + j];
      r = plot_find(P, static_cast<uint32_t>(chain[dd]), key, static_cast<uint32_t>(k));
    }
    probe[(wi * n_sub + si) * md + dd] = r;
  }
  __syncthreads();
  // ---- phase 1b: resolve_window (retrieval.cpp:23-69): for position p of the window, the
  // longest stored sub-gram containing it, leftmost among equals; first chain hit wins
  for (int t = threadIdx.x; t < n_win * n; t += blockDim.x) {
    const int wi = t / n, p = t % n;
    int start, wl;
    win_bounds(c0 + wi, start, wl);
    if (p >= wl) continue;
    int32_t row = -1, lev = 0;
    for (int k = wl; k >= 1 && row < 0; --k) {
      const int o_lo = p + 1 >= k ? p + 1 - k : 0;
      const int o_hi = p < wl - k ? p : wl - k;
      for (int o = o_lo; o <= o_hi && row < 0; ++o) {
        // sub-gram index of (o, k): sub-grams are ordered by k, then o
        const int si = (k - 1) * n - (k - 1) * (k - 2) / 2 + o;
        const int32_t* pr = &probe[(wi * n_sub + si) * md];
        for (int dd = 0; dd < depth; ++dd) {
          if (pr[dd] >= 0) {
            row = pr[dd] + (p - o);
            lev = k;
            break;
          }
        }
      }
    }
    if (row < 0) atomicExch(err, HMI_BUILD_ERROR);  // uni-gram backstop missing
    wrow[wi * n + p] = row;
    wlev[wi * n + p] = lev;
  }
  __syncthreads();

  // ---- phase 2: Eq. 2 aggregation, one warp per position
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = blockDim.x >> 5;
  const int d = P.d;
  for (int p = p0 + warp; p < p1; p += nwarps) {
    const long long orow = dec_pos ? static_cast<long long>(b) : static_cast<long long>(b) * S + p;
    int32_t rows[kMaxNgram] = {};
    int32_t levs[kMaxNgram] = {};
    int cnt = 0;
    if (p < len) {
      if (causal) {
        const int start = p + 1 >= n ? p + 1 - n : 0;
        rows[0] = wrow[(p - c0) * n + (p - start)];
        levs[0] = wlev[(p - c0) * n + (p - start)];
        cnt = 1;
      } else {
        const int c_lo = p - hr > 0 ? p - hr : 0;
        const int c_hi = p + hl < len - 1 ? p + hl : len - 1;
        for (int c = c_lo; c <= c_hi; ++c) {
          const int start = c >= hl ? c - hl : 0;
          rows[cnt] = wrow[(c - c0) * n + (p - start)];
          levs[cnt] = wlev[(c - c0) * n + (p - start)];
          ++cnt;
        }
      }
    }
    if (gather && lane < n) {
      int32_t gr = -1, gl = 0;
      for (int k = 0; k < cnt; ++k) {
        if (k == lane) { gr = rows[k]; gl = levs[k]; }
      }
      gather[orow * n + lane] = gr;
      levels[orow * n + lane] = gl;
    }
    if constexpr (V > 0) {
      gather_mean<V, NG, GV>(P.reps, rows, cnt, d, lane, orow, h16, bf16, h64);
    } else {
      const double inv = cnt > 0 ? 1.0 / static_cast<double>(cnt) : 0.0;
      for (int i = 0; i < d / 128; ++i) {
        const int col = (lane + 32 * i) * 4;
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        float4 xs[kMaxNgram];
#pragma unroll
        for (int k = 0; k < kMaxNgram; ++k) {
          if (k < cnt) {
            const int32_t r = rows[k] < 0 ? 0 : rows[k];
            xs[k] = __ldg(reinterpret_cast<const float4*>(P.reps + static_cast<long long>(r) * d + col));
          }
        }
#pragma unroll
        for (int k = 0; k < kMaxNgram; ++k) {  // ascending window order (add_f64 sweep)
          if (k < cnt) {
            a0 = a0 + static_cast<double>(xs[k].x);
            a1 = a1 + static_cast<double>(xs[k].y);
            a2 = a2 + static_cast<double>(xs[k].z);
            a3 = a3 + static_cast<double>(xs[k].w);
          }
        }
        a0 *= inv; a1 *= inv; a2 *= inv; a3 *= inv;
        if (h64) {
          double* o = h64 + orow * d + col;
          o[0] = a0; o[1] = a1; o[2] = a2; o[3] = a3;
        }
        // f64 -> f32 -> 16-bit with hardware conversions (the f64 values are the exact
        // Eq. 2 result; the 16-bit copy is the GEMM operand)
        const float f0 = __double2float_rn(a0), f1 = __double2float_rn(a1);
        const float f2 = __double2float_rn(a2), f3 = __double2float_rn(a3);
        uint2 pk;
        if (bf16) {
          pk.x = pack16x2<true>(f0, f1);
          pk.y = pack16x2<true>(f2, f3);
        } else {
          pk.x = pack16x2<false>(f0, f1);
          pk.y = pack16x2<false>(f2, f3);
        }
        *reinterpret_cast<uint2*>(static_cast<uint16_t*>(h16) + orow * d + col) = pk;
      }
    }
  }
}

__global__ void fetch_inputs_kernel(FetchArgs A) {
  const long long tid = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  const long long nthr = static_cast<long long>(gridDim.x) * blockDim.x;
  if (tid == 0 && A.d_err) *A.d_err = 0;
  const int cols = A.src_stride < A.S ? A.src_stride : A.S;
  const long long ntok = static_cast<long long>(A.n_req) * A.S;
  for (long long i = tid; i < ntok; i += nthr) {
    const long long r = i / A.S, c = i - r * A.S;
    if (c < cols) A.d_tokens[i] = A.tokens[r * A.src_stride + c];
  }
  for (long long i = tid; i < A.n_inst; i += nthr) A.d_inst[i] = A.inst[i];
  if (A.lens)
    for (long long i = tid; i < A.n_req; i += nthr) A.d_lens[i] = A.lens[i];
  for (long long i = tid; i < A.n_delta; i += nthr) A.d_delta[i] = A.delta[i];
}

// ---------------------------------------------------------------------------
// K6: routing
// ---------------------------------------------------------------------------
__global__ void route_kernel(const uint32_t* __restrict__ instance_idx, int n_req,
                             const int32_t* __restrict__ inst_version,
                             const int32_t* __restrict__ inst_task,
                             const int32_t* __restrict__ inst_head, int n_instances,
                             const int32_t* __restrict__ slot_of, int layers, int tiles_per_req,
                             int tile_stride,
                             int32_t* __restrict__ req_version, int32_t* __restrict__ req_task,
                             int32_t* __restrict__ req_head, int32_t* __restrict__ tile_slot,
                             int32_t* __restrict__ err) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_req) return;
  const uint32_t inst = instance_idx[i];
  int32_t v = -1, t = -1, h = -1;
  if (inst < static_cast<uint32_t>(n_instances)) {
    v = inst_version[inst];
    t = inst_task[inst];
    h = inst_head[inst];
  }
  if (v < 0 || t < 0 || h < 0) {
    atomicExch(err, HMI_ROUTING_ERROR);
    v = 0; t = -1; h = 0;
  }
  req_version[i] = v;
  req_task[i] = t;
  req_head[i] = h;
  for (int l = 0; l < layers; ++l) {
    int32_t s = t >= 0 ? slot_of[static_cast<long long>(t) * layers + l] : -1;
    if (s < 0) {
      atomicExch(err, HMI_SCHEDULING_BUG);  // compute reached a non-resident adapter
      s = 0;
    }
    for (int k = 0; k < tiles_per_req; ++k) tile_slot[static_cast<long long>(l) * tile_stride + i * tiles_per_req + k] = s;
  }
}

// Slot-table maintenance: table[pairs[2k]] = pairs[2k+1], applied in order.
__global__ void apply_deltas_kernel(int32_t* __restrict__ table, const int32_t* __restrict__ pairs,
                                    int n) {
  // order matters only for repeated indices; one thread keeps the host's order
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    for (int k = 0; k < n; ++k) table[pairs[2 * k]] = pairs[2 * k + 1];
  }
}

// ---------------------------------------------------------------------------
// K7: heads. cls/lm: one CTA per request over the selected row; token_tag: one
// warp per valid row. f64 accumulation of an f32 row against f32 weights.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double load16(const void* p, long long i, int bf16) {
  const uint16_t u = static_cast<const uint16_t*>(p)[i];
  if (bf16) return static_cast<double>(__uint_as_float(static_cast<uint32_t>(u) << 16));
  return static_cast<double>(__half2float(__ushort_as_half(u)));
}

// block-wide sum (all threads get the result); scratch holds blockDim doubles
__device__ __forceinline__ double block_sum(double v, double* scratch) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  __syncthreads();
  if (lane == 0) scratch[warp] = v;
  __syncthreads();
  double t = 0.0;
  for (int w = 0; w < nw; ++w) t += scratch[w];
  __syncthreads();
  return t;
}

// Final LayerNorm of pre-norm 16-bit rows from partial statistics (warp per row).
__global__ void normalize_rows_kernel(const uint16_t* __restrict__ y, const float2* __restrict__ st,
                                      int n_part, float inv_n, const float* __restrict__ g,
                                      const float* __restrict__ be, float* __restrict__ out,
                                      int rows, int d, int bf16) {
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  float s1 = 0.f, s2 = 0.f;
  for (int i = 0; i < n_part; ++i) {
    s1 += st[static_cast<long long>(row) * 16 + i].x;
    s2 += st[static_cast<long long>(row) * 16 + i].y;
  }
  const float mean = s1 * inv_n;
  const float inv = 1.0f / sqrtf(fmaxf(s2 * inv_n - mean * mean, 0.f) + 1e-5f);
  for (int j = lane; j < d; j += 32) {
    const float v = static_cast<float>(load16(y, static_cast<long long>(row) * d + j, bf16));
    out[static_cast<long long>(row) * d + j] = (v - mean) * inv * g[j] + be[j];
  }
}

__global__ void __launch_bounds__(256) head_kernel(HeadDev H, const float* __restrict__ h32,
                                                   const int32_t* __restrict__ req_head,
                                                   const int* __restrict__ lens, int S, int d,
                                                   int max_labels, float* __restrict__ scores,
                                                   int32_t* __restrict__ labels_out,
                                                   int32_t* __restrict__ tags) {
  extern __shared__ double shd[];
  const int b = blockIdx.x;
  const int hid = req_head[b];
  const int kind = H.kind[hid];
  const int nl = H.labels[hid];
  const float* W = H.arena + H.offset[hid];
  const float* B = W + static_cast<long long>(d) * nl;
  const int len = lens[b];
  if (kind == 2 && nl > max_labels) return;  // wide lm head: served by the lm GEMM path
  if (kind == 1) {
    // token_tag: rows < valid_len, argmax per row
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int r = warp; r < len; r += blockDim.x >> 5) {
      const long long rbase = (static_cast<long long>(b) * S + r) * d;
      const float* x = h32 + rbase;
      double mean = 0.0, inv = 1.0;
      if (H.y16) {  // LayerNorm of the pre-norm row, f64 (ops.cpp:92-116)
        double s1 = 0.0;
        for (int j = lane; j < d; j += 32) s1 += load16(H.y16, rbase + j, H.bf16);
        for (int o = 16; o > 0; o >>= 1) s1 += __shfl_xor_sync(0xffffffffu, s1, o);
        mean = s1 / d;
        double s2 = 0.0;
        for (int j = lane; j < d; j += 32) {
          const double t = load16(H.y16, rbase + j, H.bf16) - mean;
          s2 += t * t;
        }
        for (int o = 16; o > 0; o >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, o);
        inv = 1.0 / sqrt(s2 / d + 1e-5);
      }
      double best = -INFINITY;
      int besti = 0;
      for (int l0 = 0; l0 < nl; l0 += 32) {
        const int l = l0 + lane;
        double acc = 0.0;
        if (l < nl) {
          for (int j = 0; j < d; ++j) {
            const double xj = H.y16 ? (load16(H.y16, rbase + j, H.bf16) - mean) * inv * H.ln_g[j] + H.ln_b[j]
                                    : static_cast<double>(x[j]);
            acc += xj * W[static_cast<long long>(j) * nl + l];
          }
          acc += B[l];
        }
        // serial first-max scan over this chunk in label order (model.cpp:122-128)
        for (int k = 0; k < 32 && l0 + k < nl; ++k) {
          const double v = __shfl_sync(0xffffffffu, acc, k);
          if (v > best) { best = v; besti = l0 + k; }
        }
      }
      if (lane == 0) tags[static_cast<long long>(b) * S + r] = besti;
    }
    if (threadIdx.x == 0) labels_out[b] = -1;
    return;
  }
  const int row = kind == 0 ? 0 : len - 1;
  const long long rbase = (static_cast<long long>(b) * S + row) * d;
  const float* x = h32 + rbase;
  double* xs = shd;                       // d
  double* rv = shd + d;                   // blockDim reduction values
  int* ri = reinterpret_cast<int*>(rv + blockDim.x);
  if (H.y16) {
    // LayerNorm of the pre-norm row in f64 (ops.cpp:92-116), then the head product
    double s1 = 0.0;
    for (int j = threadIdx.x; j < d; j += blockDim.x) {
      xs[j] = load16(H.y16, rbase + j, H.bf16);
      s1 += xs[j];
    }
    const double mean = block_sum(s1, rv) / d;
    double s2 = 0.0;
    for (int j = threadIdx.x; j < d; j += blockDim.x) {
      const double t = xs[j] - mean;
      s2 += t * t;
    }
    const double inv = 1.0 / sqrt(block_sum(s2, rv) / d + 1e-5);
    for (int j = threadIdx.x; j < d; j += blockDim.x)
      xs[j] = (xs[j] - mean) * inv * H.ln_g[j] + H.ln_b[j];
  } else {
    for (int j = threadIdx.x; j < d; j += blockDim.x) xs[j] = x[j];
  }
  __syncthreads();
  double best = -INFINITY;
  int besti = 0x7fffffff;
  if (nl <= 32) {
    // narrow head (cls): split d across the block, reduce per label
    double acc[32];
#pragma unroll
    for (int l = 0; l < 32; ++l) acc[l] = 0.0;
    for (int j = threadIdx.x; j < d; j += blockDim.x) {
      const double xj = xs[j];
      const float* wr = W + static_cast<long long>(j) * nl;
#pragma unroll
      for (int l = 0; l < 32; ++l)
        if (l < nl) acc[l] += xj * static_cast<double>(__ldg(wr + l));
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
#pragma unroll
    for (int l = 0; l < 32; ++l) {
      if (l >= nl) break;
      double v = acc[l];
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) rv[warp * 32 + l] = v;  // rv has room for blockDim doubles
    }
    __syncthreads();
    if (threadIdx.x < nl) {
      const int l = threadIdx.x;
      double s = 0.0;
      for (int w = 0; w < nw; ++w) s += rv[w * 32 + l];
      s += static_cast<double>(B[l]);
      if (l < max_labels) scores[static_cast<long long>(b) * max_labels + l] = static_cast<float>(s);
      best = s;
      besti = l;
    }
    __syncthreads();
  } else {
    // wide head (lm): one label per thread, W rows read coalesced across the block
    for (int l = threadIdx.x; l < nl; l += blockDim.x) {
      double acc = 0.0;
      for (int j = 0; j < d; ++j) acc += xs[j] * static_cast<double>(W[static_cast<long long>(j) * nl + l]);
      acc += static_cast<double>(B[l]);
      if (l < max_labels) scores[static_cast<long long>(b) * max_labels + l] = static_cast<float>(acc);
      if (acc > best) { best = acc; besti = l; }  // labels visited in ascending order
    }
  }
  rv[threadIdx.x] = best;
  ri[threadIdx.x] = besti;
  __syncthreads();
  for (int off = blockDim.x / 2; off > 0; off >>= 1) {
    if (threadIdx.x < off) {
      const double ov = rv[threadIdx.x + off];
      const int oi = ri[threadIdx.x + off];
      // first max (model.cpp:122-128): larger value wins, ties go to the lower index
      if (ov > rv[threadIdx.x] || (ov == rv[threadIdx.x] && oi < ri[threadIdx.x])) {
        rv[threadIdx.x] = ov;
        ri[threadIdx.x] = oi;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) labels_out[b] = ri[0] == 0x7fffffff ? 0 : ri[0];
}

}  // namespace

void launch_layernorm(const float* y, const float* gamma, const float* beta, void* out16,
                      float* out32, int rows, int d, int precision, cudaStream_t stream,
                      int n_parts, long long part_stride, const float* bias, const void* res16_) {
  const auto* res16 = static_cast<const uint16_t*>(res16_);
  if (rows <= 0) return;
  HMI_CHECK(d % 128 == 0 && d <= 2048, HMI_CONFIG_ERROR, "layernorm: d must be a multiple of 128");
  const int blocks = (rows + 7) / 8;
  auto* o16 = static_cast<uint16_t*>(out16);
#define HMI_LN_CASE(VV)                                                                       \
  case VV:                                                                                    \
    if (precision == 1)                                                                       \
      layernorm_kernel<VV, true><<<blocks, 256, 0, stream>>>(y, gamma, beta, o16, out32, rows, n_parts, part_stride, bias, res16); \
    else                                                                                      \
      layernorm_kernel<VV, false><<<blocks, 256, 0, stream>>>(y, gamma, beta, o16, out32, rows, n_parts, part_stride, bias, res16); \
    break;
  switch (d / 128) {
    HMI_LN_CASE(1) HMI_LN_CASE(2) HMI_LN_CASE(3) HMI_LN_CASE(4) HMI_LN_CASE(5) HMI_LN_CASE(6)
    HMI_LN_CASE(7) HMI_LN_CASE(8) HMI_LN_CASE(9) HMI_LN_CASE(10) HMI_LN_CASE(11)
    HMI_LN_CASE(12) HMI_LN_CASE(13) HMI_LN_CASE(14) HMI_LN_CASE(15) HMI_LN_CASE(16)
    default: break;
  }
#undef HMI_LN_CASE
  HMI_CUDA(cudaGetLastError());
}

void launch_retrieve(const PlotDev& plot, const uint32_t* tokens, const int* lens,
                     const int* req_version, int n_req, int S, int causal, void* h16,
                     int precision, double* h64_debug, int32_t* gather, int32_t* levels,
                     int32_t* err, cudaStream_t stream, const int32_t* dec_pos, int tok_stride) {
  if (n_req <= 0) return;
  HMI_CHECK(plot.d % 128 == 0, HMI_CONFIG_ERROR, "retrieve: d must be a multiple of 128");
  HMI_CHECK(!dec_pos || causal, HMI_CONFIG_ERROR, "retrieve: decode rows need causal mode");
  dim3 grid(n_req, dec_pos ? 1 : (S + kRetrieveChunk - 1) / kRetrieveChunk);
  const int n = plot.ngram;
  const size_t smem = static_cast<size_t>(kRetrieveChunk + kMaxNgram) * (n * (n + 1) / 2) *
                      plot.max_depth * sizeof(int32_t);
  // phase 2 specialised for the hidden sizes of BASELINE's configs (d = 256 / 768 / 1024) and
  // the window count per position (encoder: n windows; causal: 1): two float4 columns of every
  // row in flight per lane at 5 CTAs per SM (C2 in-step 107 -> 82 us; all six columns in flight
  // at 2 CTAs per SM: 126 us, one column at 6 CTAs: 88 us, three at 4: 96 us — same box)
  const int V = plot.d / 128;
  const int NG = causal ? 1 : plot.ngram;
  auto go = [&](auto kern) {
    kern<<<grid, 256, smem, stream>>>(plot, tokens, lens, req_version, S, causal, h16, precision,
                                      h64_debug, gather, levels, err, dec_pos, tok_stride);
  };
#define HMI_RETR_CASE(VV, NN)                   \
  if (V == VV && NG == NN) {                    \
    go(retrieve_kernel<VV, NN, 2, 5>);          \
    HMI_CUDA(cudaGetLastError());               \
    return;                                     \
  }
  HMI_RETR_CASE(6, 3) HMI_RETR_CASE(6, 1) HMI_RETR_CASE(8, 3) HMI_RETR_CASE(8, 1)
  HMI_RETR_CASE(2, 3) HMI_RETR_CASE(2, 1)
#undef HMI_RETR_CASE
  go(retrieve_kernel<0, kMaxNgram, 1, 6>);
  HMI_CUDA(cudaGetLastError());
}

void launch_route(const uint32_t* instance_idx, int n_req, const int32_t* inst_version,
                  const int32_t* inst_task, const int32_t* inst_head, int n_instances,
                  const int32_t* slot_of, int layers, int tiles_per_req, int tile_stride,
                  int32_t* req_version, int32_t* req_task, int32_t* req_head,
                  int32_t* tile_slot, int32_t* err, cudaStream_t stream) {
  if (n_req <= 0) return;
  route_kernel<<<(n_req + 127) / 128, 128, 0, stream>>>(
      instance_idx, n_req, inst_version, inst_task, inst_head, n_instances, slot_of, layers,
      tiles_per_req, tile_stride, req_version, req_task, req_head, tile_slot, err);
  HMI_CUDA(cudaGetLastError());
}

void launch_normalize_rows(const void* y16, const float2* stats, int n_part, float inv_n,
                           const float* gamma, const float* beta, float* out, int rows, int d,
                           int precision, cudaStream_t stream) {
  if (rows <= 0) return;
  normalize_rows_kernel<<<(rows + 7) / 8, 256, 0, stream>>>(
      static_cast<const uint16_t*>(y16), stats, n_part, inv_n, gamma, beta, out, rows, d,
      precision);
  HMI_CUDA(cudaGetLastError());
}

void launch_fetch_inputs(const FetchArgs& a, cudaStream_t stream) {
  const long long work = static_cast<long long>(a.n_req) * a.S;
  const int blocks = static_cast<int>(std::min<long long>((work + 255) / 256 + 1, 4 * device_sm_count()));
  fetch_inputs_kernel<<<blocks, 256, 0, stream>>>(a);
  HMI_CUDA(cudaGetLastError());
}

// One warp per entry: its rows are contiguous f32 in the raw chunk (4-byte aligned: PLT1 entry
// sizes are multiples of 4) and contiguous in the reps arena.
__global__ void scatter_rows_kernel(const uint8_t* __restrict__ chunk, const int4* __restrict__ segs,
                                    int n_seg, float* __restrict__ dst, int d) {
  const int lane = threadIdx.x & 31;
  const int nwarps = static_cast<int>(gridDim.x * blockDim.x >> 5);
  for (int s = static_cast<int>((blockIdx.x * blockDim.x + threadIdx.x) >> 5); s < n_seg; s += nwarps) {
    const int4 g = segs[s];
    const float* in = reinterpret_cast<const float*>(chunk + g.x);
    float* out = dst + ((static_cast<size_t>(g.y) | (static_cast<size_t>(g.z) << 31)) * d);
    const int n = g.w * d;
    for (int i = lane; i < n; i += 32) out[i] = in[i];
  }
}

void launch_scatter_rows(const uint8_t* chunk, const int4* segs, int n_seg, float* dst, int d,
                         cudaStream_t stream) {
  if (n_seg <= 0) return;
  const int blocks = std::min((n_seg + 7) / 8, 8 * device_sm_count());
  scatter_rows_kernel<<<blocks, 256, 0, stream>>>(chunk, segs, n_seg, dst, d);
  HMI_CUDA(cudaGetLastError());
}

void launch_apply_deltas(int32_t* table, const int32_t* pairs, int n, cudaStream_t stream) {
  if (n <= 0) return;
  apply_deltas_kernel<<<1, 32, 0, stream>>>(table, pairs, n);
  HMI_CUDA(cudaGetLastError());
}

void launch_head(const HeadDev& heads, const float* h32, const int32_t* req_head,
                 const int* lens, int n_req, int S, int d, int max_labels, float* scores,
                 int32_t* labels_out, int32_t* tags, cudaStream_t stream) {
  if (n_req <= 0) return;
  const size_t smem = static_cast<size_t>(d + 256) * sizeof(double) + 256 * sizeof(int);
  if (smem > 48 * 1024) {
    HMI_CUDA(cudaFuncSetAttribute(head_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
  }
  head_kernel<<<n_req, 256, smem, stream>>>(heads, h32, req_head, lens, S, d, max_labels, scores,
                                            labels_out, tags);
  HMI_CUDA(cudaGetLastError());
}

}  // namespace hmi_b200
