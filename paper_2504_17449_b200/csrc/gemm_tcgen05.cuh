// SPDX-License-Identifier: Apache-2.0
//
// K1/K2 — persistent, warp-specialised tcgen05 GEMM for sm_100a.
//
//   C[M x N] = epilogue( A[M x K] . B^T )   A: 16-bit row-major (K-major)
//                                           B: 16-bit [groups][N][K]   (K-major, 3-D TMA map)
//
// Replaces every `gemm_f64` call on the hot path (proj/src/tensor/kernels_scalar.cpp:11-26
// via matmul_into, proj/src/tensor/ops.cpp:25-36):
//   * attention Q/K/V and output projections (proj/src/transformer/model.cpp:35-37, :75)
//   * FFN (model.cpp:78-82) with the bias+ReLU epilogue fused
//   * the tenant-grouped adapter products (proj/src/adapters/stacked.cpp:44-64) — "grouped"
//     mode: every 128-row M tile belongs to exactly one request, and the B tile is
//     gathered from that request's HBM slot (tile_slot[m_tile] selects the group).
//
// Roles (320 threads, 1 CTA per SM):
//   warp 0      : TMA producer (one elected lane)      smem ring of kStages (A,B) tiles
//   warp 1      : TMEM allocator + MMA issuer (lane 0)  2 TMEM accumulators of BN fp32 cols
//   warps 2..9  : epilogue, TMEM -> regs -> bias/ReLU/residual -> 16/32-bit -> smem -> TMA store
#pragma once

#include "gemm.hpp"
#include "sm100.cuh"

namespace hmi_b200 {

constexpr int kGemmThreads = 320;  // TMA warp, MMA warp, 8 epilogue warps
constexpr int kBlockM = 128;
constexpr int kBlockK = 64;  // 64 x 16-bit = 128 B = one SWIZZLE_128B atom row


template <bool kBf16>
__device__ __forceinline__ uint32_t pack_16x2(float a, float b) {
  if constexpr (kBf16) {
    const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<const uint32_t*>(&h);
  } else {
    const __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<const uint32_t*>(&h);
  }
}

// v[0..32) += 32 16-bit residuals of one row of a SWIZZLE_128B smem box, starting at
// 16-byte chunk ch0 of the row (row base `rowp`, rsw = row % 8)
template <bool kBf16>
__device__ __forceinline__ void add_res16_smem(float* v, const uint8_t* rowp, int ch0, int rsw) {
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const uint4 u = *reinterpret_cast<const uint4*>(rowp + (((ch0 + k) ^ rsw) << 4));
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      float2 f;
      if constexpr (kBf16) {
        f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[e]));
      } else {
        f = __half22float2(*reinterpret_cast<const __half2*>(&w[e]));
      }
      v[8 * k + 2 * e] += f.x;
      v[8 * k + 2 * e + 1] += f.y;
    }
  }
}

// v[0..N) += 16-bit residual row segment (16-byte vector loads)
template <bool kBf16, int N>
__device__ __forceinline__ void add_res16(float* v, const uint16_t* src) {
#pragma unroll
  for (int i = 0; i < N; i += 8) {
    const uint4 u = __ldg(reinterpret_cast<const uint4*>(src + i));
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      float2 f;
      if constexpr (kBf16) {
        f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[e]));
      } else {
        f = __half22float2(*reinterpret_cast<const __half2*>(&w[e]));
      }
      v[i + 2 * e] += f.x;
      v[i + 2 * e + 1] += f.y;
    }
  }
}

// Row (mean, 1/sqrt(var + eps)) of a pre-norm row from P partial (sum, sumsq) entries
// (layer_norm, ops.cpp:92-116: biased variance, epsilon 1e-5).
__device__ __forceinline__ float2 row_stats(const float2* part, int n, float inv_n) {
  // all partials in one round trip: kStatsStride float2 = 8 x 16-byte loads (rows are 128 B)
  float4 q[kStatsStride / 2];
#pragma unroll
  for (int i = 0; i < kStatsStride / 2; ++i) {
    q[i] = 2 * i < n ? __ldg(reinterpret_cast<const float4*>(part) + i) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  float s1 = 0.f, s2 = 0.f;
#pragma unroll
  for (int i = 0; i < kStatsStride / 2; ++i) {
    s1 += q[i].x;
    s2 += q[i].y;
    if (2 * i + 1 < n) {
      s1 += q[i].z;
      s2 += q[i].w;
    }
  }
  const float mean = s1 * inv_n;
  const float var = fmaxf(s2 * inv_n - mean * mean, 0.0f);
  return make_float2(mean, 1.0f / sqrtf(var + 1e-5f));
}

// v[0..N) += LN(pre-norm 16-bit residual row segment): (y - mean) * inv * gamma + beta
template <bool kBf16, int N>
__device__ __forceinline__ void add_res16_ln(float* v, const uint16_t* src, float2 st,
                                             const float* gamma, const float* beta) {
  float r[N];
#pragma unroll
  for (int i = 0; i < N; ++i) r[i] = 0.f;
  add_res16<kBf16, N>(r, src);
#pragma unroll
  for (int i = 0; i < N; i += 4) {
    const float4 g = __ldg(reinterpret_cast<const float4*>(gamma + i));
    const float4 b = __ldg(reinterpret_cast<const float4*>(beta + i));
    v[i] += (r[i] - st.x) * st.y * g.x + b.x;
    v[i + 1] += (r[i + 1] - st.x) * st.y * g.y + b.y;
    v[i + 2] += (r[i + 2] - st.x) * st.y * g.z + b.z;
    v[i + 3] += (r[i + 3] - st.x) * st.y * g.w + b.w;
  }
}

// r[0..N) = 16-bit residuals of (row_local, columns c..c+N) from TMA-staged SWIZZLE_128B
// boxes [BN/64][128 rows][128 B]
template <bool kBf16, int N>
__device__ __forceinline__ void res_from_smem(float* r, const uint8_t* boxes, int row_local,
                                              int c) {
#pragma unroll
  for (int i = 0; i < N; ++i) r[i] = 0.f;
#pragma unroll
  for (int i = 0; i < N; i += 32) {
    const uint8_t* rowp = boxes + ((c + i) >> 6) * 16384 + row_local * 128;
    add_res16_smem<kBf16>(r + i, rowp, ((c + i) & 63) >> 3, row_local & 7);
  }
}

// v += r, or v += LN(r) = (r - mean) * inv * gamma + beta
template <int N, bool kLn>
__device__ __forceinline__ void add_res_vals(float* v, const float* r, float2 st,
                                             const float* gamma, const float* beta) {
  if constexpr (kLn) {
#pragma unroll
    for (int i = 0; i < N; i += 4) {
      const float4 g = __ldg(reinterpret_cast<const float4*>(gamma + i));
      const float4 b = __ldg(reinterpret_cast<const float4*>(beta + i));
      v[i] += (r[i] - st.x) * st.y * g.x + b.x;
      v[i + 1] += (r[i + 1] - st.x) * st.y * g.y + b.y;
      v[i + 2] += (r[i + 2] - st.x) * st.y * g.z + b.z;
      v[i + 3] += (r[i + 3] - st.x) * st.y * g.w + b.w;
    }
  } else {
#pragma unroll
    for (int i = 0; i < N; ++i) v[i] += r[i];
  }
}

// Partial-statistics row of the one LN input an epilogue folds (A's for kEpiFoldLN, the
// residual's for kEpiRes{0,1}LN), loaded a unit ahead so its latency is off the epilogue's path.
template <int EPI>
struct StatsPrefetch {
  static constexpr bool kA = (EPI & kEpiFoldLN) != 0;
  static constexpr bool kR = (EPI & (kEpiRes0LN | kEpiRes1LN)) != 0;
  static_assert(!(kA && kR), "one folded LayerNorm input per epilogue");
  float4 q[kStatsStride / 2];
  __device__ __forceinline__ void load(const GemmArgs& args, int row) {
    if constexpr (kA || kR) {
      const float2* part = (kA ? args.a_stats : args.r_stats) + static_cast<long long>(row) * kStatsStride;
      const int n = kA ? args.a_stats_n : args.r_stats_n;
#pragma unroll
      for (int i = 0; i < kStatsStride / 2; ++i) {
        q[i] = row < args.M && 2 * i < n ? __ldg(reinterpret_cast<const float4*>(part) + i)
                                         : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
  }
  // (mean, 1 / sqrt(var + eps)) into a_st or r_st
  __device__ __forceinline__ void finish(const GemmArgs& args, float2& a_st, float2& r_st) const {
    a_st = make_float2(0.f, 1.f);
    r_st = make_float2(0.f, 1.f);
    if constexpr (kA || kR) {
      float s1 = 0.f, s2 = 0.f;
#pragma unroll
      for (int i = 0; i < kStatsStride / 2; ++i) {  // entries beyond n were loaded as zero
        s1 += q[i].x + q[i].z;
        s2 += q[i].y + q[i].w;
      }
      const float mean = s1 * args.inv_n;
      const float var = fmaxf(s2 * args.inv_n - mean * mean, 0.0f);
      const float2 st = make_float2(mean, 1.0f / sqrtf(var + 1e-5f));
      if constexpr (kA) a_st = st; else r_st = st;
    }
  }
};

// Row statistics the LN-folding epilogue modes need (fetched before the accumulator wait)
template <int EPI>
__device__ __forceinline__ void epi_row_stats(const GemmArgs& args, int mt, uint32_t q,
                                              uint32_t lane, float2& a_st, float2& r_st) {
  a_st = make_float2(0.f, 1.f);
  r_st = make_float2(0.f, 1.f);
  const int row = mt * kBlockM + static_cast<int>(q) * 32 + static_cast<int>(lane);
  if (row >= args.M) return;
  if constexpr ((EPI & kEpiFoldLN) != 0) {
    a_st = row_stats(args.a_stats + static_cast<long long>(row) * kStatsStride, args.a_stats_n,
                     args.inv_n);
  }
  if constexpr ((EPI & (kEpiRes0LN | kEpiRes1LN)) != 0) {
    r_st = row_stats(args.r_stats + static_cast<long long>(row) * kStatsStride, args.r_stats_n,
                     args.inv_n);
  }
}

// One accumulator tile (128 rows x BN cols in TMEM) -> bias / residual / ReLU -> 16/32-bit
// -> swizzled smem staging -> TMA store. Called by 8 epilogue warps: warp (q, half) owns TMEM
// lane quarter q and every other kCW-column chunk.
// LayerNorm folding: kEpiFoldLN rescales the accumulator of a pre-norm A operand by its
// row statistics; kEpiRes{0,1}LN normalise a pre-norm residual on the fly; kEpiStats
// emits this thread's partial row (sum, sumsq) for the next consumer.
//
// kStaged (pair kernel, one 16-bit residual): this warp's k-th chunk of the tile has its
// residual box (32 rows x 64 columns) TMA-loaded into staging buffer k, completing on
// rbar[k] (parity bit k of rph); the output is written back over it and stored from there.
// kSVec: the unit's column vectors come from shared memory: svec[0, BN) bias (+ the tenant
// bias), [BN, 2 BN) LN gamma and [2 BN, 3 BN) LN beta of the residual, or colsum (kEpiFoldLN).
template <int BN, int EPI, bool kStaged = false, bool kSVec = false, int kBufs = 2>
__device__ __forceinline__ void epilogue_tile(uint32_t t_acc, int mt, int col_base, int ncols,
                                              int grp, const GemmArgs& args,
                                              const CUtensorMap* map_c, uint8_t* stg,
                                              uint32_t& sbuf, uint32_t q, int half,
                                              uint32_t lane, float2 a_st, float2 r_st,
                                              const uint8_t* res_smem, uint64_t* rbar = nullptr,
                                              uint32_t* rph = nullptr,
                                              const float* svec = nullptr) {
  constexpr bool kResTma = (EPI & kEpiResTma) != 0;  // residual tiles staged in smem by TMA
  constexpr bool kOutF32 = (EPI & kEpiOutF32) != 0;
  constexpr bool kBf16 = (EPI & kEpiBf16) != 0;  // 16-bit tensors are bf16 (else fp16)
  constexpr int kCW = kOutF32 ? 32 : 64;         // output columns per 128-byte staging row
  static_assert(BN % kCW == 0, "BN must be a multiple of the store chunk");
  static_assert((EPI & kEpiStats) == 0 || !kOutF32, "row statistics need 16-bit outputs");
  const float* bias = args.bias + grp * args.bias_slot_stride + col_base;
  const int row0 = mt * kBlockM + static_cast<int>(q) * 32;
  const int row = row0 + static_cast<int>(lane);
  const bool row_ok = row < args.M;
  const uint32_t t_row = t_acc + ((q * 32) << 16);
  static_assert(!kStaged || (!kOutF32 && (EPI & kEpiRes1) != 0 && (EPI & kEpiRes2) == 0),
                "staged residuals: one 16-bit residual, 16-bit output");
  int kc = 0;  // this warp's chunk index within the tile (kStaged: its staging buffer)
#pragma unroll 1
  for (int c = half * kCW; c < ncols; c += 2 * kCW, ++kc) {
    float v[kCW];
    {
      uint32_t r[kCW];  // both TMEM loads in flight, one wait
#pragma unroll
      for (int j = 0; j < kCW / 32; ++j) {
        tmem_ld_32x32b_x32(t_row + c + 32 * j, *reinterpret_cast<uint32_t(*)[32]>(r + 32 * j));
      }
      tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < kCW; ++i) v[i] = __uint_as_float(r[i]);
    }
    if constexpr ((EPI & kEpiFoldLN) != 0) {
      const float* cs = args.colsum + col_base + c;
#pragma unroll
      for (int i = 0; i < kCW; i += 4) {
        const float4 c4 = kSVec ? *reinterpret_cast<const float4*>(svec + BN + c + i)
                                : __ldg(reinterpret_cast<const float4*>(cs + i));
        v[i] = a_st.y * (v[i] - a_st.x * c4.x);
        v[i + 1] = a_st.y * (v[i + 1] - a_st.x * c4.y);
        v[i + 2] = a_st.y * (v[i + 2] - a_st.x * c4.z);
        v[i + 3] = a_st.y * (v[i + 3] - a_st.x * c4.w);
      }
    }
    if constexpr (kSVec) {
#pragma unroll
      for (int i = 0; i < kCW; i += 4) {
        const float4 b4 = *reinterpret_cast<const float4*>(svec + c + i);
        v[i] += b4.x; v[i + 1] += b4.y; v[i + 2] += b4.z; v[i + 3] += b4.w;
      }
    } else {
#pragma unroll
      for (int i = 0; i < kCW; i += 4) {
        const float4 b4 = __ldg(reinterpret_cast<const float4*>(bias + c + i));
        v[i] += b4.x; v[i + 1] += b4.y; v[i + 2] += b4.z; v[i + 3] += b4.w;
      }
    }
    if constexpr (!kSVec && (EPI & kEpiExt) != 0) {  // the tile's tenant bias (b_u of its slot)
      const float* b2 = args.bias2 + grp * args.bias2_stride + col_base + c;
#pragma unroll
      for (int i = 0; i < kCW; i += 4) {
        const float4 b4 = __ldg(reinterpret_cast<const float4*>(b2 + i));
        v[i] += b4.x; v[i + 1] += b4.y; v[i + 2] += b4.z; v[i + 3] += b4.w;
      }
    }
    if constexpr (kStaged) {
      if (row0 < args.M) {  // else nothing was staged: the rows are past the batch
        mbar_wait(&rbar[kc], (*rph >> kc) & 1u);
        *rph ^= 1u << kc;
      }
      const uint8_t* rowp = stg + kc * 4096 + lane * 128;
#pragma unroll
      for (int k = 0; k < 8; ++k) {  // 16-byte chunks, consumed as they are read
        const uint4 u = *reinterpret_cast<const uint4*>(rowp + ((k ^ (lane & 7)) << 4));
        const uint32_t w[4] = {u.x, u.y, u.z, u.w};
        float f[8];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          float2 t;
          if constexpr (kBf16) {
            t = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[e]));
          } else {
            t = __half22float2(*reinterpret_cast<const __half2*>(&w[e]));
          }
          f[2 * e] = t.x;
          f[2 * e + 1] = t.y;
        }
        if constexpr ((EPI & kEpiRes0LN) != 0) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const float4 g = *reinterpret_cast<const float4*>(svec + BN + c + 8 * k + 4 * h);
            const float4 b = *reinterpret_cast<const float4*>(svec + 2 * BN + c + 8 * k + 4 * h);
            float* vv = v + 8 * k + 4 * h;
            const float* ff = f + 4 * h;
            vv[0] += (ff[0] - r_st.x) * r_st.y * g.x + b.x;
            vv[1] += (ff[1] - r_st.x) * r_st.y * g.y + b.y;
            vv[2] += (ff[2] - r_st.x) * r_st.y * g.z + b.z;
            vv[3] += (ff[3] - r_st.x) * r_st.y * g.w + b.w;
          }
        } else {
#pragma unroll
          for (int e = 0; e < 8; ++e) v[8 * k + e] += f[e];
        }
      }
    } else if constexpr ((EPI & (kEpiRes1 | kEpiRes2)) != 0) {
      const int col = col_base + c;
      if constexpr (kResTma) {
        const int row_local = static_cast<int>(q) * 32 + static_cast<int>(lane);
        float r[kCW];
        res_from_smem<kBf16, kCW>(r, res_smem, row_local, c);
        add_res_vals<kCW, (EPI & kEpiRes0LN) != 0>(v, r, r_st, args.r_gamma + col,
                                                   args.r_beta + col);
        if constexpr ((EPI & kEpiRes2) != 0) {
          res_from_smem<kBf16, kCW>(r, res_smem + (BN / 64) * 16384, row_local, c);
          add_res_vals<kCW, (EPI & kEpiRes1LN) != 0>(v, r, r_st, args.r_gamma + col,
                                                     args.r_beta + col);
        }
      } else if (row_ok) {
        const long long off = static_cast<long long>(row) * args.res_ld + col;
        if constexpr ((EPI & kEpiRes0LN) != 0) {
          add_res16_ln<kBf16, kCW>(v, reinterpret_cast<const uint16_t*>(args.res0) + off, r_st,
                                   args.r_gamma + col, args.r_beta + col);
        } else {
          add_res16<kBf16, kCW>(v, reinterpret_cast<const uint16_t*>(args.res0) + off);
        }
        if constexpr ((EPI & kEpiRes2) != 0) {
          if constexpr ((EPI & kEpiRes1LN) != 0) {
            add_res16_ln<kBf16, kCW>(v, reinterpret_cast<const uint16_t*>(args.res1) + off, r_st,
                                     args.r_gamma + col, args.r_beta + col);
          } else {
            add_res16<kBf16, kCW>(v, reinterpret_cast<const uint16_t*>(args.res1) + off);
          }
        }
      }
    }
    if constexpr ((EPI & kEpiRelu) != 0) {
#pragma unroll
      for (int i = 0; i < kCW; ++i) v[i] = fmaxf(v[i], 0.0f);
    }
    if constexpr ((EPI & kEpiStats) != 0) {  // partial of this 64-column group
      float s1 = 0.f, s2 = 0.f;
#pragma unroll
      for (int i = 0; i < kCW; ++i) {
        s1 += v[i];
        s2 += v[i] * v[i];
      }
      if (row_ok) {
        args.stats_out[static_cast<long long>(row) * args.stats_ld + (col_base + c) / 64] =
            make_float2(s1, s2);
      }
    }
    uint32_t packed[32];  // one 128-byte row per thread
    if constexpr (kOutF32) {
#pragma unroll
      for (int i = 0; i < 32; ++i) packed[i] = __float_as_uint(v[i]);
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i) packed[i] = pack_16x2<kBf16>(v[2 * i], v[2 * i + 1]);
    }
    uint8_t* buf;
    if constexpr (kStaged) {
      buf = stg + kc * 4096;  // over this chunk's residual (each thread rewrites its own row)
    } else {
      // double-buffered staging: the store issued from this buffer two chunks ago is read
      if (lane == 0) tma_store_wait_read<kBufs - 1>();
      __syncwarp();
      buf = stg + sbuf * 4096;
      sbuf = (sbuf + 1) % kBufs;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int phys = i ^ (lane & 7);  // SWIZZLE_128B: 16 B chunk ^= row % 8
      *reinterpret_cast<uint4*>(buf + lane * 128 + phys * 16) =
          make_uint4(packed[4 * i], packed[4 * i + 1], packed[4 * i + 2], packed[4 * i + 3]);
    }
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0 && mt < args.num_m_tiles) {
      tma_store_2d(map_c, buf, col_base + c, row0);
      tma_store_commit();
    }
  }
}

// Fine pipeline: block until the copy stream has published this layer's adapter slots
// (*ready reaches ready_seq, written by cuStreamWriteValue32 after the layer's H2D copies), so
// a stream-level event wait does not cut the programmatic-launch chain. Whole CTA.
__device__ __forceinline__ void wait_ready(const GemmArgs& args) {
  if (args.ready == nullptr) return;
  if (threadIdx.x == 0) {
    const uint64_t t0 = globaltimer_ns();
    while (ld_acquire_gpu(args.ready) - args.ready_seq > 0x7fffffffu) {  // wrap-safe <
      if (globaltimer_ns() - t0 > 20ull * 1000 * 1000 * 1000) {  // 20 s: never, unless broken
        atomicExch(args.err, HMI_SCHEDULING_BUG);
        break;
      }
      __nanosleep(256);
    }
    fence_proxy_async_global();  // the slots are read through TMA (async proxy)
  }
  __syncthreads();
}

template <int BN, bool RT = false>
struct GemmSmem {
  static constexpr int kABytes = kBlockM * kBlockK * 2;  // 16 KB
  static constexpr int kBBytes = BN * kBlockK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  // 8 epilogue warps x (32 rows x 128 B), double-buffered except with staged residuals and
  // at BN = 64 (one store per warp and tile: the space goes to ring stages instead)
  static constexpr bool kSingleStg = RT || BN == 64;
  static constexpr int kEpiBytes = kSingleStg ? 8 * 4096 : 8 * 2 * 4096;
  // RT: two residual tiles of 128 rows x BN (BN/64 SWIZZLE_128B boxes of 16 KB each)
  static constexpr int kResBytes = RT ? 2 * (BN / 64) * 16384 : 0;
  static constexpr int kBudget = 227 * 1024 - 1024 /*align*/ - 256 /*barriers*/;
  static constexpr int kStagesRaw = (kBudget - kEpiBytes - kResBytes) / kStageBytes;
  static constexpr int kStagesCap = RT ? 2 : 8;  // RT GEMMs have a single K block (K = r)
  static constexpr int kStages = kStagesRaw > kStagesCap ? kStagesCap : kStagesRaw;
  static constexpr int kTotal =
      1024 + kStages * kStageBytes + kEpiBytes + kResBytes + 256;
  static constexpr int kTmemCols = 2 * BN <= 32 ? 32 : 2 * BN <= 64 ? 64 : 2 * BN <= 128 ? 128
                                 : 2 * BN <= 256 ? 256 : 512;
};

template <int BN, int EPI>
__global__ void __launch_bounds__(kGemmThreads, 1)
    gemm_tcgen05_kernel(const __grid_constant__ GemmMaps maps, const GemmArgs args) {
  const CUtensorMap& map_a = maps.a;
  const CUtensorMap& map_b = maps.b;
  const CUtensorMap& map_c = maps.c;
  constexpr bool kRT = (EPI & kEpiResTma) != 0;
  using L = GemmSmem<BN, kRT>;
  constexpr int kStages = L::kStages;
  static_assert(kStages >= 2, "smem budget too small");
  static_assert(BN % 32 == 0 && BN >= 32 && BN <= 256, "BN");

  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + ((1024 - (raw_addr & 1023)) & 1023);
  uint8_t* sA = smem;
  uint8_t* sB = smem + kStages * L::kABytes;
  uint8_t* sEpi = smem + kStages * L::kStageBytes;
  uint8_t* sRes = sEpi + L::kEpiBytes;  // kRT only
  uint64_t* bars = reinterpret_cast<uint64_t*>(sRes + L::kResBytes);
  uint64_t* full = bars;
  uint64_t* empty = bars + kStages;
  uint64_t* tfull = bars + 2 * kStages;
  uint64_t* tempty = bars + 2 * kStages + 2;
  uint64_t* res_full = bars + 2 * kStages + 6;   // kRT
  uint64_t* res_empty = bars + 2 * kStages + 7;  // kRT
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kStages + 8);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const int num_tiles = args.num_m_tiles * args.num_n_tiles;
  const int num_kb = args.K / kBlockK;
  // tile schedule: persistent grid-stride
  const int t_first = blockIdx.x, t_step = gridDim.x;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&map_a);
    tma_prefetch_desc(&map_b);
    tma_prefetch_desc(&map_c);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 8);
    }
    if constexpr (kRT) {
      mbar_init(res_full, 1);
      mbar_init(res_empty, 8);
      tma_prefetch_desc(&maps.r0);
      tma_prefetch_desc(&maps.r1);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<L::kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_trigger();
  pdl_wait();  // inputs of the previous kernel are complete and visible from here on
  wait_ready(args);

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      const uint64_t pol_a = policy_evict_first();
      const uint64_t pol_b = policy_evict_last();
      uint32_t stage = 0, phase = 0, res_phase = 0;
      for (int t = t_first; t < num_tiles; t += t_step) {
        const int mt = t / args.num_n_tiles;
        const int nt = t - mt * args.num_n_tiles;
        const int grp = args.tile_slot ? __ldg(&args.tile_slot[mt]) : 0;
        if constexpr (kRT) {
          // residual tiles for this tile's epilogue (single buffer, released after pass 1)
          mbar_wait(res_empty, res_phase ^ 1);
          constexpr int nbox = BN / 64;
          mbar_arrive_expect_tx(res_full, 2 * nbox * 16384);
          for (int j = 0; j < nbox; ++j) {
            tma_load_2d(sRes + j * 16384, &maps.r0, res_full, nt * BN + j * 64, mt * kBlockM);
            tma_load_2d(sRes + (nbox + j) * 16384, &maps.r1, res_full, nt * BN + j * 64,
                        mt * kBlockM);
          }
          res_phase ^= 1;
        }
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full[stage], L::kStageBytes);
          tma_load_2d_hint(sA + stage * L::kABytes, &map_a, &full[stage], kb * kBlockK,
                           mt * kBlockM, pol_a);
          tma_load_3d_hint(sB + stage * L::kBBytes, &map_b, &full[stage], kb * kBlockK,
                           nt * BN, grp, pol_b);
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      uint32_t stage = 0, phase = 0, acc = 0, acc_phase = 0;
      for (int t = t_first; t < num_tiles; t += t_step) {
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint64_t a_desc = sdesc_k_sw128(smem_u32(sA + stage * L::kABytes));
          const uint64_t b_desc = sdesc_k_sw128(smem_u32(sB + stage * L::kBBytes));
#pragma unroll
          for (int k = 0; k < kBlockK / 16; ++k) {
            // +32 B along K inside the 128 B swizzle atom = +2 in the 16 B address field
            umma_f16(d_tmem, a_desc + 2 * k, b_desc + 2 * k, args.idesc, (kb | k) != 0);
          }
          umma_commit(&empty[stage]);
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
        umma_commit(&tfull[acc]);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const uint32_t q = warp & 3;  // TMEM lane quarter this warp may access
    const int half = static_cast<int>(warp - 2) >> 2;
    uint8_t* stg = sEpi + (warp - 2) * (L::kSingleStg ? 4096 : 2 * 4096);
    uint32_t sbuf = 0;
    uint32_t acc = 0, acc_phase = 0, iter = 0;
    for (int t = t_first; t < num_tiles; t += t_step, ++iter) {
      const int mt = t / args.num_n_tiles;
      const int nt = t - mt * args.num_n_tiles;
      const int grp = args.tile_slot ? __ldg(&args.tile_slot[mt]) : 0;
      float2 a_st, r_st;
      epi_row_stats<EPI>(args, mt, q, lane, a_st, r_st);
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      if constexpr (kRT) mbar_wait(res_full, iter & 1);
      epilogue_tile<BN, EPI, false, false, L::kSingleStg ? 1 : 2>(tmem_base + acc * BN, mt, nt * BN, BN, grp, args, &map_c, stg, sbuf,
                             q, half, lane, a_st, r_st, sRes);
      if constexpr (kRT) {  // residual tiles consumed: the producer may stage the next tile's
        __syncwarp();
        if (lane == 0) mbar_arrive(res_empty);
      }
      // all TMEM reads of this accumulator by this warp are done: hand it back
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
    if (lane == 0) tma_store_wait_all<0>();
    __syncwarp();
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<L::kTmemCols>(tmem_base);
  }
}

// ===========================================================================
// cta_group::2 variant for the shared-weight GEMMs: a CTA pair (cluster of 2)
// computes a 256 x BN tile with UMMA M = 256. Each CTA TMA-loads its own 128
// rows of A and half (BN/2 rows) of the B tile into its own smem, crediting the
// leader's (rank 0) full barrier; the leader's single MMA thread issues
// tcgen05.mma.cta_group::2 reading A and B from both CTAs, so per SM the smem
// operand traffic per MMA is A/2 + B/2 of the 1-CTA kernel's. Commits multicast
// to both CTAs' empty / tmem-full barriers; both CTAs' epilogues drain their
// own 128 TMEM lanes and arrive on the leader's tmem-empty barrier.
// ===========================================================================
// Pair-kernel work unit v: a 256 x BN tile, or (in the wave tail) one of tail_split
// sub-tiles of width BN / tail_split.
struct PairUnit {
  int mp, col0, width;
  bool tail;
};

template <int BN>
__device__ __forceinline__ PairUnit pair_unit(const GemmArgs& a, int v) {
  PairUnit p;
  int u = v, sub = 0;
  p.tail = a.tail_split > 1 && v >= a.n_main;
  if (p.tail) {
    const int t = v - a.n_main;
    u = a.n_main + t / a.tail_split;
    sub = t - (t / a.tail_split) * a.tail_split;
  }
  p.mp = u / a.num_n_tiles;
  const int nt = u - p.mp * a.num_n_tiles;
  p.width = p.tail ? BN / a.tail_split : BN;
  p.col0 = nt * BN + sub * p.width;
  return p;
}

__device__ __forceinline__ int pair_units_total(const GemmArgs& a, int num_units) {
  return a.tail_split > 1 ? a.n_main + (num_units - a.n_main) * a.tail_split : num_units;
}

// Pair-kernel epilogues with one 16-bit residual and a 16-bit output stage that residual by
// TMA through the epilogue buffers; they and the LN-folding epilogues read the unit's column
// vectors from shared memory.
constexpr bool pair_staged(int epi) {
  return (epi & kEpiRes1) != 0 && (epi & (kEpiRes2 | kEpiOutF32)) == 0;
}
constexpr bool pair_svec(int epi) { return pair_staged(epi); }

template <int BN, bool kVec = false>
struct Gemm2Smem {
  static constexpr int kABytes = kBlockM * kBlockK * 2;          // this CTA's 128 rows of A
  static constexpr int kBBytes = (BN / 2) * kBlockK * 2;         // this CTA's half of B
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kEpiBytes = 8 * 2 * 4096;  // 8 epilogue warps x 2 staging buffers
  static constexpr int kVecBytes = kVec ? 2 * 3 * BN * 4 : 0;    // two units' column vectors
  static constexpr int kBarBytes = 512;  // ring, accumulator and staged-residual barriers
  static constexpr int kBudget = 227 * 1024 - 1024 - kBarBytes;
  static constexpr int kStagesRaw = (kBudget - kEpiBytes - kVecBytes) / kStageBytes;
  static constexpr int kStages = kStagesRaw > 8 ? 8 : kStagesRaw;
  static constexpr int kTotal = 1024 + kStages * kStageBytes + kEpiBytes + kVecBytes + kBarBytes;
  static constexpr int kTmemCols = 2 * BN <= 256 ? 256 : 512;
};

template <int BN, int EPI>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kGemmThreads, 1)
    gemm2_tcgen05_kernel(const __grid_constant__ GemmMaps maps, const GemmArgs args) {
  const CUtensorMap& map_a = maps.a;
  const CUtensorMap& map_b = maps.b;
  const CUtensorMap& map_c = maps.c;
  constexpr bool kStaged = pair_staged(EPI);
  constexpr bool kSVec = pair_svec(EPI);
  using L = Gemm2Smem<BN, kSVec>;
  constexpr int kStages = L::kStages;
  static_assert(kStages >= 3, "smem budget too small");
  static_assert(BN % 32 == 0 && BN >= 64 && BN <= 256, "BN");

  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + ((1024 - (raw_addr & 1023)) & 1023);
  uint8_t* sA = smem;
  uint8_t* sB = smem + kStages * L::kABytes;
  uint8_t* sEpi = smem + kStages * L::kStageBytes;
  float* sVec = reinterpret_cast<float*>(sEpi + L::kEpiBytes);  // kSVec: [2][3][BN]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sEpi + L::kEpiBytes + L::kVecBytes);
  uint64_t* full = bars;
  uint64_t* empty = bars + kStages;
  uint64_t* tfull = bars + 2 * kStages;
  uint64_t* tempty = bars + 2 * kStages + 2;
  uint64_t* rbars = bars + 2 * kStages + 4;  // [8 epilogue warps][2] staged residual boxes
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kStages + 20);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const uint32_t rank = cluster_ctarank();
  const int n_pairs = (args.num_m_tiles + 1) / 2;
  const int num_units = n_pairs * args.num_n_tiles;
  const int total = pair_units_total(args, num_units);
  const int cluster = blockIdx.x >> 1;
  const int n_clusters = gridDim.x >> 1;
  constexpr bool kExt = (EPI & kEpiExt) != 0;
  const int num_kb = args.K / kBlockK;
  const int all_kb = num_kb + (kExt ? 2 * args.ext_kb : 0);

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&map_a);
    tma_prefetch_desc(&map_b);
    tma_prefetch_desc(&map_c);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 16);  // 8 epilogue warps x 2 CTAs (leader's copy is the one used)
    }
    for (int s = 0; s < 16; ++s) mbar_init(&rbars[s], 1);
    if constexpr (kStaged) tma_prefetch_desc(&maps.res);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc_2cta<L::kTmemCols>(tmem_slot);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_trigger();
  // pdl_wait (the previous kernel complete and visible) per role: the producer first stages
  // the shared weights of its first ring lap, which no kernel writes, then waits; the MMA
  // thread touches no global memory; the epilogue waits before its first read

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer (both CTAs)
    if (lane == 0) {
      const uint64_t pol_a = policy_evict_first();
      const uint64_t pol_b = policy_evict_last();
      uint32_t stage = 0, phase = 0;
      // first ring lap: B (shared weights) of the first unit's first stages before pdl_wait
      int pre = 0;
      if (cluster < total) {
        const PairUnit pu = pair_unit<BN>(args, cluster);
        const CUtensorMap* mb = !pu.tail ? &map_b : args.tail_r1 ? &maps.r1 : &maps.r0;
        const uint32_t bytes = 2 * (L::kABytes + (pu.width / 2) * kBlockK * 2);
        const int col = pu.col0 + static_cast<int>(rank) * (pu.width / 2);
        pre = num_kb < kStages ? num_kb : kStages;
        for (int kb = 0; kb < pre; ++kb) {
          if (rank == 0) mbar_arrive_expect_tx(&full[kb], bytes);
          tma_load_3d_2sm(sB + kb * L::kBBytes, mb, mapa_shared(smem_u32(&full[kb]), 0),
                          kb * kBlockK, col, 0, pol_b);
        }
      }
      pdl_wait();
      for (int v = cluster; v < total; v += n_clusters) {
        const PairUnit pu = pair_unit<BN>(args, v);
        const int mt = 2 * pu.mp + static_cast<int>(rank);
        // wave-tail sub-tiles load B through the narrower-box maps r0 / r1
        const CUtensorMap* mb = !pu.tail ? &map_b : args.tail_r1 ? &maps.r1 : &maps.r0;
        const uint32_t bytes = 2 * (L::kABytes + (pu.width / 2) * kBlockK * 2);
        for (int kb = 0; kb < all_kb; ++kb) {
          const bool staged_b = pre > 0;  // this stage's B went out before pdl_wait
          if (!staged_b) {
            mbar_wait(&empty[stage], phase ^ 1);
            if (rank == 0) mbar_arrive_expect_tx(&full[stage], bytes);
          }
          const uint32_t leader_full = mapa_shared(smem_u32(&full[stage]), 0);
          const int col = pu.col0 + static_cast<int>(rank) * (pu.width / 2);
          if (!kExt || kb < num_kb) {
            tma_load_2d_2sm(sA + stage * L::kABytes, &map_a, leader_full, kb * kBlockK,
                            mt * kBlockM, pol_a);
            if (!staged_b) {
              tma_load_3d_2sm(sB + stage * L::kBBytes, mb, leader_full, kb * kBlockK, col, 0, pol_b);
            } else {
              --pre;
            }
          } else {
            // tenant block: tile e's ext rows against tile e's slot; the other CTA's A half
            // is the zero rows, so rows of the other request gain nothing
            const int x = kb - num_kb;
            const int e = x / args.ext_kb, kx = (x - e * args.ext_kb) * kBlockK;
            const int mte = 2 * pu.mp + e;
            const int slot = mte < args.num_m_tiles ? __ldg(&args.tile_slot[mte]) : 0;
            const CUtensorMap* xb = !pu.tail ? &maps.xb : args.tail_r1 ? &maps.xb1 : &maps.xb0;
            tma_load_2d_2sm(sA + stage * L::kABytes, &maps.xa, leader_full, kx,
                            e == static_cast<int>(rank) ? mt * kBlockM : args.ext_zero_row, pol_a);
            tma_load_3d_2sm(sB + stage * L::kBBytes, xb, leader_full, kx, col, slot, pol_b);
          }
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (leader only)
    if (rank == 0 && lane == 0) {
      uint32_t stage = 0, phase = 0, acc = 0, acc_phase = 0;
      for (int v = cluster; v < total; v += n_clusters) {
        const uint32_t idesc = args.tail_split > 1 && v >= args.n_main ? args.idesc_tail : args.idesc;
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < all_kb; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint64_t a_desc = sdesc_k_sw128(smem_u32(sA + stage * L::kABytes));
          const uint64_t b_desc = sdesc_k_sw128(smem_u32(sB + stage * L::kBBytes));
#pragma unroll
          for (int k = 0; k < kBlockK / 16; ++k) {
            umma_f16_2cta(d_tmem, a_desc + 2 * k, b_desc + 2 * k, idesc, (kb | k) != 0);
          }
          umma_commit_2cta_mc(&empty[stage], 0x3);
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
        umma_commit_2cta_mc(&tfull[acc], 0x3);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue (both CTAs)
    pdl_wait();
    const uint32_t q = warp & 3;
    const int half = static_cast<int>(warp - 2) >> 2;
    uint8_t* stg = sEpi + (warp - 2) * 2 * 4096;
    uint64_t* rbar = rbars + (warp - 2) * 2;
    uint32_t sbuf = 0, rph = 0;
    uint32_t acc = 0, acc_phase = 0;
    // kStaged: residual boxes of unit v's chunks for this warp (32 rows x 64 columns each)
    // into its two staging buffers, once the stores issued from them have read them
    StatsPrefetch<EPI> spf;
    auto fetch_stats = [&](int v) {
      if (v >= total) return;
      const PairUnit pn = pair_unit<BN>(args, v);
      spf.load(args, (2 * pn.mp + static_cast<int>(rank)) * kBlockM + static_cast<int>(q) * 32 +
                         static_cast<int>(lane));
    };
    fetch_stats(cluster);
    auto stage_res = [&](int v) {
      if (v >= total) return;
      const PairUnit pn = pair_unit<BN>(args, v);
      const int row0 = (2 * pn.mp + static_cast<int>(rank)) * kBlockM + static_cast<int>(q) * 32;
      if (row0 >= args.M) return;  // rows past the batch (odd tile count): nothing to stage
      tma_store_wait_read<0>();
      int k = 0;
      for (int c = half * 64; c < pn.width; c += 128, ++k) {
        mbar_arrive_expect_tx(&rbar[k], 4096);
        tma_load_2d(stg + k * 4096, &maps.res, &rbar[k], pn.col0 + c, row0);
      }
    };
    if constexpr (kStaged) {
      if (lane == 0) stage_res(cluster);
    }
    uint32_t iter = 0;
    for (int v = cluster; v < total; v += n_clusters, ++iter) {
      const PairUnit pu = pair_unit<BN>(args, v);
      const int mt = 2 * pu.mp + static_cast<int>(rank);
      const int grp = kExt && mt < args.num_m_tiles ? __ldg(&args.tile_slot[mt]) : 0;
      float* sv = sVec + (iter & 1) * 3 * BN;
      if constexpr (kSVec) {
        // this unit's column vectors, one column per epilogue thread; the buffer written here
        // was last read two units ago, before every warp passed the previous unit's barrier
        const int t = static_cast<int>(warp - 2) * 32 + static_cast<int>(lane);
        if (t < pu.width) {
          const int col = pu.col0 + t;
          float b = __ldg(args.bias + col);
          if constexpr (kExt) b += __ldg(args.bias2 + grp * args.bias2_stride + col);
          sv[t] = b;
          if constexpr ((EPI & kEpiRes0LN) != 0) {
            sv[BN + t] = __ldg(args.r_gamma + col);
            sv[2 * BN + t] = __ldg(args.r_beta + col);
          }
          if constexpr ((EPI & kEpiFoldLN) != 0) sv[BN + t] = __ldg(args.colsum + col);
        }
        named_bar_sync(1, 256);
      }
      float2 a_st, r_st;
      spf.finish(args, a_st, r_st);
      fetch_stats(v + n_clusters);
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      epilogue_tile<BN, EPI, kStaged, kSVec>(tmem_base + acc * BN, mt, pu.col0, pu.width, grp, args,
                                      &map_c, stg, sbuf, q, half, lane, a_st, r_st, nullptr, rbar,
                                      &rph, sv);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(mapa_shared(smem_u32(&tempty[acc]), 0));
      if constexpr (kStaged) {
        if (lane == 0) stage_res(v + n_clusters);
      }
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
    if (lane == 0) tma_store_wait_all<0>();
    __syncwarp();
  }

  tc_fence_before();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_2cta<L::kTmemCols>(tmem_base);
  }
}

}  // namespace hmi_b200
