// SPDX-License-Identifier: Apache-2.0
//
// K3 on the 5th-gen tensor cores, padded length 128 (the hBERT / hGPT serving shape).
//
// Same math as attention() (proj/src/transformer/model.cpp:39-74): per (request, head)
// S = Q K^T / sqrt(64) over keys j < limit (valid_len, or i + 1 when causal), softmax,
// ctx = P V. One persistent CTA per SM walks (request, head) items, double-buffered:
//
//   warp 0 (lane 0): TMA   Q, K, V tiles (128 x 64 16-bit, SWIZZLE_128B) -> smem stage
//                          (kStages items in flight)
//   warp 1 (lane 0): MMA   S[buf] = Q K^T   tcgen05 M=128 N=128 K=64 -> TMEM; issued one item
//                          ahead of O[buf] = P V (M=128 N=64 K=128, V as MN-major B), so the
//                          two softmax groups run concurrently
//   warps 2..9     : softmax, two groups of 4 warps (group g serves buffer g, i.e. every
//                    other item, so two items' softmax overlap); one query row per
//                    thread: TMEM S row -> mask / max / exp2 / sum -> 16-bit P row into
//                    swizzled smem over the consumed Q, K tiles (UMMA A operand); epilogue: TMEM O row * 1/sum ->
//                    16-bit -> smem -> TMA store
//
// Barriers per load stage: load_full (TMA tx), load_empty (MMA commit after P.V); per TMEM
// buffer: s_full (MMA commit), p_full (4 softmax warps), o_full (MMA commit), o_empty (4 warps).
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <cstdint>

#include "kernels.hpp"
#include "sm100.cuh"

namespace hmi_b200 {

namespace {

constexpr int kTcThreads = 320;  // TMA warp, MMA warp, 2 groups x 4 softmax warps
constexpr int kT = 128 * 128;                // one 128 x 64 16-bit tile (bytes)
constexpr int kStages = 4;                   // Q, K, V load stages (items in flight)
constexpr int kBufBytes = 3 * kT;            // Q, K, V; P (128 x 128 16-bit) overwrites Q, K
constexpr int kOStage = kT;                  // output staging tile
constexpr int kSmem = 1024 + kStages * kBufBytes + 2 * kOStage + 256;

// Shared-memory descriptor of an MN-major SWIZZLE_128B operand whose MN extent is one
// 128-byte atom (64 x 16-bit): 8-row K groups are 1024 B apart.
__device__ __forceinline__ uint64_t sdesc_mn_sw128(uint32_t smem_addr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((smem_addr & 0x3FFFFu) >> 4);
  d |= static_cast<uint64_t>(8192 >> 4) << 16;  // LBO: next MN atom (unused, N = 64)
  d |= static_cast<uint64_t>(1024 >> 4) << 32;  // SBO: next 8 K rows
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(2) << 61;
  return d;
}

__device__ __forceinline__ uint32_t sw(int r, int chunk) {
  return static_cast<uint32_t>(r * 128 + ((chunk ^ (r & 7)) << 4));
}

// 2^x on the MUFU (ex2.approx.ftz: denormal results flush to zero; softmax weights that small
// vanish against the row's maximum term, which is exactly 1)
__device__ __forceinline__ float ex2_ftz(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

template <bool kBf16>
__device__ __forceinline__ uint32_t pk2(float a, float b) {
  if constexpr (kBf16) {
    const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<const uint32_t*>(&h);
  } else {
    const __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<const uint32_t*>(&h);
  }
}

template <bool kBf16>
__global__ void __launch_bounds__(kTcThreads, 1) attention_tc_kernel(
    const __grid_constant__ CUtensorMap map_qkv, const __grid_constant__ CUtensorMap map_ctx,
    const int* __restrict__ lens, int n_items, int heads, int d, int causal, float scale_log2) {
  extern __shared__ uint8_t raw[];
  uint8_t* base = raw + ((1024 - (smem_u32(raw) & 1023)) & 1023);
  uint8_t* ostg = base + kStages * kBufBytes;
  uint64_t* bar = reinterpret_cast<uint64_t*>(ostg + 2 * kOStage);
  uint64_t* load_full = bar;                  // [kStages]
  uint64_t* load_empty = bar + kStages;       // [kStages]
  uint64_t* s_full = bar + 2 * kStages;       // [2]
  uint64_t* p_full = s_full + 2;              // [2]
  uint64_t* o_full = s_full + 4;              // [2]
  uint64_t* o_empty = s_full + 6;             // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(s_full + 8);

  const uint32_t warp = warp_id(), lane = lane_id();
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&map_qkv);
    tma_prefetch_desc(&map_ctx);
    for (int b = 0; b < kStages; ++b) {
      mbar_init(&load_full[b], 1);
      mbar_init(&load_empty[b], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&s_full[b], 1);
      mbar_init(&p_full[b], 4);
      mbar_init(&o_full[b], 1);
      mbar_init(&o_empty[b], 4);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_trigger();
  pdl_wait();
  // TMEM columns: S[0] 0..127, S[1] 128..255, O[0] 256..319, O[1] 320..383
  const int my_first = blockIdx.x, step = gridDim.x;

  if (warp == 0) {
    if (lane == 0) {
      int k = 0;
      for (int item = my_first; item < n_items; item += step, ++k) {
        const int b = k % kStages;
        const uint32_t ph = (k / kStages) & 1;
        mbar_wait(&load_empty[b], ph ^ 1);
        const int req = item / heads, h = item - req * heads;
        uint8_t* dst = base + b * kBufBytes;
        mbar_arrive_expect_tx(&load_full[b], 3 * kT);
        tma_load_2d(dst, &map_qkv, &load_full[b], h * 64, req * 128);
        tma_load_2d(dst + kT, &map_qkv, &load_full[b], d + h * 64, req * 128);
        tma_load_2d(dst + 2 * kT, &map_qkv, &load_full[b], 2 * d + h * 64, req * 128);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t id_s = idesc_f16(128, 128, kBf16 ? 1u : 0u);
      const uint32_t id_o = idesc_f16(128, 64, kBf16 ? 1u : 0u) | (1u << 16);  // B MN-major
      const int n_mine = my_first < n_items ? (n_items - 1 - my_first) / step + 1 : 0;
      auto issue_s = [&](int k) {  // S[k & 1] = Q K^T of this CTA's k-th item
        const int st = k % kStages;
        mbar_wait(&load_full[st], (k / kStages) & 1);
        tc_fence_after();
        uint8_t* buf = base + st * kBufBytes;
        const uint64_t qd = sdesc_k_sw128(smem_u32(buf));
        const uint64_t kd = sdesc_k_sw128(smem_u32(buf + kT));
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {  // K = 64 = 4 x 16; +32 B inside the swizzle atom per step
          umma_f16(tmem + (k & 1) * 128, qd + 2 * kk, kd + 2 * kk, id_s, kk);
        }
        umma_commit(&s_full[k & 1]);
      };
      if (n_mine > 0) issue_s(0);
      for (int k = 0; k < n_mine; ++k) {
        const int b = k & 1;
        const uint32_t ph = (k >> 1) & 1;
        // S of the next item first: its TMEM buffer was released by p_full(k - 1), waited below
        // in the previous iteration, so both softmax groups have work
        if (k + 1 < n_mine) issue_s(k + 1);
        // O[b] = P V once the softmax wrote P and the epilogue released O[b]
        mbar_wait(&p_full[b], ph);
        mbar_wait(&o_empty[b], ph ^ 1);
        tc_fence_after();
        uint8_t* buf = base + (k % kStages) * kBufBytes;
        const uint32_t p0 = smem_u32(buf), vb = smem_u32(buf + 2 * kT);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {  // 16 keys per step
          const uint64_t pd = sdesc_k_sw128(p0 + (kk >> 2) * kT) + 2 * (kk & 3);
          const uint64_t vd = sdesc_mn_sw128(vb + kk * 2048);
          umma_f16(tmem + 256 + b * 64, pd, vd, id_o, kk);
        }
        umma_commit(&o_full[b]);
        umma_commit(&load_empty[k % kStages]);  // Q, K, V, P of this stage consumed
      }
    }
  } else {
    const uint32_t q = warp & 3;      // TMEM lane quarter
    const int group = static_cast<int>(warp - 2) >> 2;  // serves buffer `group`
    uint8_t* gstg = ostg + group * kOStage;
    const int r = static_cast<int>(q * 32 + lane);  // query row owned by this thread
    const uint32_t lane_off = (q * 32) << 16;
    float l_prev = 0.f;
    int prev_item = -1, prev_b = 0;
    uint32_t prev_ph = 0;
    auto epilogue = [&](int item, int b, uint32_t ph, float l) {
      mbar_wait(&o_full[b], ph);
      tc_fence_after();
      uint32_t o[64];
      tmem_ld_32x32b_x32(tmem + lane_off + 256 + b * 64, *reinterpret_cast<uint32_t(*)[32]>(o));
      tmem_ld_32x32b_x32(tmem + lane_off + 256 + b * 64 + 32,
                         *reinterpret_cast<uint32_t(*)[32]>(o + 32));
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&o_empty[b]);
      const float inv = l > 0.f ? 1.f / l : 0.f;
      // the staging tile is free once the previous item's store has read it; only the
      // thread that issued that store can wait on it
      if (q == 0 && lane == 0) tma_store_wait_read<0>();
      named_bar_sync(1 + group, 128);
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        uint4 v;
        v.x = pk2<kBf16>(__uint_as_float(o[8 * c + 0]) * inv, __uint_as_float(o[8 * c + 1]) * inv);
        v.y = pk2<kBf16>(__uint_as_float(o[8 * c + 2]) * inv, __uint_as_float(o[8 * c + 3]) * inv);
        v.z = pk2<kBf16>(__uint_as_float(o[8 * c + 4]) * inv, __uint_as_float(o[8 * c + 5]) * inv);
        v.w = pk2<kBf16>(__uint_as_float(o[8 * c + 6]) * inv, __uint_as_float(o[8 * c + 7]) * inv);
        *reinterpret_cast<uint4*>(gstg + sw(r, c)) = v;
      }
      fence_proxy_async_smem();
      named_bar_sync(1 + group, 128);
      if (q == 0 && lane == 0) {
        const int req = item / heads, h = item - req * heads;
        tma_store_2d(&map_ctx, gstg, h * 64, req * 128);
        tma_store_commit();
      }
    };
    int k = group;
    for (int item = my_first + group * step; item < n_items; item += 2 * step, k += 2) {
      const int b = k & 1;  // == group
      const uint32_t ph = (k >> 1) & 1;
      const int req = item / heads;
      const int valid = __ldg(&lens[req]);
      const int lim = causal ? r + 1 : valid;
      mbar_wait(&s_full[b], ph);
      tc_fence_after();
      float s[128];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        uint32_t t[32];
        tmem_ld_32x32b_x32(tmem + lane_off + b * 128 + 32 * j, t);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i) s[32 * j + i] = __uint_as_float(t[i]);
      }
      // scale (+ mask keys j >= lim: skipped, model.cpp:48-51), max and sum with four
      // independent partial chains; exp2 on the MUFU without the denormal fix-up
      float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
      if (lim >= 128) {
#pragma unroll
        for (int j = 0; j < 128; ++j) {
          s[j] *= scale_log2;
          m4[j & 3] = fmaxf(m4[j & 3], s[j]);
        }
      } else {
#pragma unroll
        for (int j = 0; j < 128; ++j) {
          s[j] = j < lim ? s[j] * scale_log2 : -INFINITY;
          m4[j & 3] = fmaxf(m4[j & 3], s[j]);
        }
      }
      const float mx = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]));
      const float mb = mx == -INFINITY ? 0.f : mx;
      float l4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int j = 0; j < 128; ++j) {
        s[j] = ex2_ftz(s[j] - mb);
        l4[j & 3] += s[j];
      }
      const float l = (l4[0] + l4[1]) + (l4[2] + l4[3]);
      // P row r -> two SWIZZLE_128B K-major tiles (keys 0-63, 64-127) over the stage's Q, K
      // (both consumed: s_full committed after the S MMA read them)
      uint8_t* P = base + (k % kStages) * kBufBytes;
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        uint4 v;
        v.x = pk2<kBf16>(s[8 * c + 0], s[8 * c + 1]);
        v.y = pk2<kBf16>(s[8 * c + 2], s[8 * c + 3]);
        v.z = pk2<kBf16>(s[8 * c + 4], s[8 * c + 5]);
        v.w = pk2<kBf16>(s[8 * c + 6], s[8 * c + 7]);
        *reinterpret_cast<uint4*>(P + (c >> 3) * kT + sw(r, c & 7)) = v;
      }
      fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[b]);
      // the previous item's output is ready by now (its P.V ran while we did this softmax)
      if (prev_item >= 0) epilogue(prev_item, prev_b, prev_ph, l_prev);
      prev_item = item;
      prev_b = b;
      prev_ph = ph;
      l_prev = l;
    }
    if (prev_item >= 0) epilogue(prev_item, prev_b, prev_ph, l_prev);
    if (q == 0 && lane == 0) tma_store_wait_all<0>();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// ---------------------------------------------------------------------------
// Padded lengths 256..512 (2..4 key blocks of 128) on tcgen05. One work item = (request,
// head, 128-query block); the item's Q, every K and V block sit in shared memory. Two passes
// over the key blocks share two TMEM score buffers: pass 1 takes the row maximum over the
// keys the reference reads (j < limit, model.cpp:48-56), pass 2 recomputes each score block,
// writes P = exp2(s - max) as 16-bit into one of two smem P buffers and accumulates
// O += P V in TMEM, then O / sum is stored. Same arithmetic as the padded-128 kernel above.
//
//   warp 0 (lane 0): TMA   Q, K[0..nb), V[0..nb) of an item (one stage)
//   warp 1 (lane 0): MMA   S(t) for t = 0 .. 2 nb - 1 into TMEM buffer t % 2, PV(j) behind
//   warps 2..5     : one query row per thread: max pass, exp / sum / P pass, epilogue
constexpr int kLThreads = 192;
constexpr int kLMaxBlocks = 4;
constexpr int kLSmem = 1024 + kT /*Q*/ + 2 * kLMaxBlocks * kT /*K, V*/ + 2 * 2 * kT /*P[2]*/ +
                       kT /*O staging*/ + 256;

template <bool kBf16>
__global__ void __launch_bounds__(kLThreads, 1) attention_long_kernel(
    const __grid_constant__ CUtensorMap map_qkv, const __grid_constant__ CUtensorMap map_ctx,
    const int* __restrict__ lens, int n_items, int heads, int nb, int d, int causal,
    float scale_log2) {
  extern __shared__ uint8_t raw[];
  uint8_t* base = raw + ((1024 - (smem_u32(raw) & 1023)) & 1023);
  uint8_t* sQ = base;
  uint8_t* sK = sQ + kT;                            // [kLMaxBlocks] 128 keys x 64
  uint8_t* sV = sK + kLMaxBlocks * kT;              // [kLMaxBlocks]
  uint8_t* sP = sV + kLMaxBlocks * kT;              // [2] 128 rows x 128 keys (two 64-key tiles)
  uint8_t* sO = sP + 4 * kT;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sO + kT);
  uint64_t* ld_full = bar;        // item operands landed (TMA tx)
  uint64_t* ld_empty = bar + 1;   // item operands consumed (MMA commit)
  uint64_t* s_full = bar + 2;     // [2] score buffer written (MMA commit)
  uint64_t* s_empty = bar + 4;    // [2] score buffer read (4 warps)
  uint64_t* p_full = bar + 6;     // [2] P buffer written (4 warps)
  uint64_t* p_empty = bar + 8;    // [2] P buffer read by the PV MMA (commit)
  uint64_t* o_full = bar + 10;    // O complete (commit)
  uint64_t* o_empty = bar + 11;   // O read (4 warps)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 12);

  const uint32_t warp = warp_id(), lane = lane_id();
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&map_qkv);
    tma_prefetch_desc(&map_ctx);
    mbar_init(ld_full, 1);
    mbar_init(ld_empty, 1);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&s_full[b], 1);
      mbar_init(&s_empty[b], 4);
      mbar_init(&p_full[b], 4);
      mbar_init(&p_empty[b], 1);
    }
    mbar_init(o_full, 1);
    mbar_init(o_empty, 4);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_trigger();
  pdl_wait();
  // TMEM columns: S buffers 0..127 and 128..255, O 256..319
  const int S = nb * 128;

  if (warp == 0) {
    if (lane == 0) {
      uint32_t ph = 0;
      for (int item = blockIdx.x; item < n_items; item += gridDim.x, ph ^= 1) {
        const int qb = item % nb, rh = item / nb, h = rh % heads, req = rh / heads;
        mbar_wait(ld_empty, ph ^ 1);
        mbar_arrive_expect_tx(ld_full, (1 + 2 * nb) * kT);
        const int row0 = req * S;
        tma_load_2d(sQ, &map_qkv, ld_full, h * 64, row0 + qb * 128);
        for (int j = 0; j < nb; ++j) {
          tma_load_2d(sK + j * kT, &map_qkv, ld_full, d + h * 64, row0 + j * 128);
          tma_load_2d(sV + j * kT, &map_qkv, ld_full, 2 * d + h * 64, row0 + j * 128);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t id_s = idesc_f16(128, 128, kBf16 ? 1u : 0u);
      const uint32_t id_o = idesc_f16(128, 64, kBf16 ? 1u : 0u) | (1u << 16);  // B MN-major
      uint32_t ld_ph = 0, o_ph = 0, s_use[2] = {0, 0}, p_use[2] = {0, 0};
      const uint64_t qd = sdesc_k_sw128(smem_u32(sQ));
      auto pv = [&](int j) {
        const int b = j & 1;
        mbar_wait(&p_full[b], p_use[b] & 1);
        ++p_use[b];
        tc_fence_after();
        const uint32_t p0 = smem_u32(sP + b * 2 * kT), vb = smem_u32(sV + j * kT);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {  // 16 keys per step
          const uint64_t pd = sdesc_k_sw128(p0 + (kk >> 2) * kT) + 2 * (kk & 3);
          const uint64_t vd = sdesc_mn_sw128(vb + kk * 2048);
          umma_f16(tmem + 256, pd, vd, id_o, (j | kk) != 0);
        }
        umma_commit(&p_empty[b]);
      };
      for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
        mbar_wait(ld_full, ld_ph);
        ld_ph ^= 1;
        tc_fence_after();
        for (int t = 0; t < 2 * nb; ++t) {
          const int b = t & 1;
          mbar_wait(&s_empty[b], (s_use[b] & 1) ^ 1);
          ++s_use[b];
          tc_fence_after();
          const uint64_t kd = sdesc_k_sw128(smem_u32(sK + (t % nb) * kT));
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) umma_f16(tmem + b * 128, qd + 2 * kk, kd + 2 * kk, id_s, kk);
          umma_commit(&s_full[b]);
          if (t == nb) {  // first PV of the item: the previous item's O has been read
            mbar_wait(o_empty, o_ph ^ 1);
            o_ph ^= 1;
          }
          if (t > nb) pv(t - nb - 1);
        }
        pv(nb - 1);
        umma_commit(o_full);
        umma_commit(ld_empty);  // Q, K, V of this item consumed
      }
    }
  } else {
    const uint32_t q = warp & 3;                    // TMEM lane quarter
    const int r = static_cast<int>(q * 32 + lane);  // query row of the block
    const uint32_t lane_off = (q * 32) << 16;
    uint32_t s_use[2] = {0, 0}, p_use[2] = {0, 0}, o_ph = 0;
    const bool storer = warp == 2 && lane == 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
      const int qb = item % nb, rh = item / nb, h = rh % heads, req = rh / heads;
      const int valid = __ldg(&lens[req]);
      const int lim = causal ? qb * 128 + r + 1 : valid;  // keys j < lim (model.cpp:48-51)
      auto read_s = [&](int t, float (&sv)[128]) {
        const int b = t & 1;
        mbar_wait(&s_full[b], s_use[b] & 1);
        ++s_use[b];
        tc_fence_after();
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t u[32];
          tmem_ld_32x32b_x32(tmem + lane_off + b * 128 + 32 * c, u);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) sv[32 * c + i] = __uint_as_float(u[i]);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&s_empty[b]);
      };
      float mx = -INFINITY;
      for (int t = 0; t < nb; ++t) {  // pass 1: row maximum of the scaled scores
        float sv[128];
        read_s(t, sv);
        const int kl = lim - t * 128;  // keys of this block below the limit
        float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
        for (int c = 0; c < 128; ++c) m4[c & 3] = fmaxf(m4[c & 3], c < kl ? sv[c] * scale_log2 : -INFINITY);
        mx = fmaxf(mx, fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3])));
      }
      const float mb = mx == -INFINITY ? 0.f : mx;
      float l4[4] = {0.f, 0.f, 0.f, 0.f};
      for (int j = 0; j < nb; ++j) {  // pass 2: P blocks and their sum
        float sv[128];
        read_s(nb + j, sv);
        const int kl = lim - j * 128;
#pragma unroll
        for (int c = 0; c < 128; ++c) {
          sv[c] = c < kl ? ex2_ftz(sv[c] * scale_log2 - mb) : 0.f;
          l4[c & 3] += sv[c];
        }
        const int b = j & 1;
        mbar_wait(&p_empty[b], (p_use[b] & 1) ^ 1);  // the PV two blocks back read this buffer
        ++p_use[b];
        uint8_t* P = sP + b * 2 * kT;
#pragma unroll
        for (int c = 0; c < 16; ++c) {
          uint4 v;
          v.x = pk2<kBf16>(sv[8 * c + 0], sv[8 * c + 1]);
          v.y = pk2<kBf16>(sv[8 * c + 2], sv[8 * c + 3]);
          v.z = pk2<kBf16>(sv[8 * c + 4], sv[8 * c + 5]);
          v.w = pk2<kBf16>(sv[8 * c + 6], sv[8 * c + 7]);
          *reinterpret_cast<uint4*>(P + (c >> 3) * kT + sw(r, c & 7)) = v;
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[b]);
      }
      const float l = (l4[0] + l4[1]) + (l4[2] + l4[3]);
      // epilogue: O / l -> 16-bit -> staging -> TMA store
      mbar_wait(o_full, o_ph);
      o_ph ^= 1;
      tc_fence_after();
      uint32_t o[64];
      tmem_ld_32x32b_x32(tmem + lane_off + 256, *reinterpret_cast<uint32_t(*)[32]>(o));
      tmem_ld_32x32b_x32(tmem + lane_off + 256 + 32, *reinterpret_cast<uint32_t(*)[32]>(o + 32));
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(o_empty);
      const float inv = l > 0.f ? 1.f / l : 0.f;
      if (storer) tma_store_wait_read<0>();  // the previous item's store has read the staging
      named_bar_sync(1, 128);
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        uint4 v;
        v.x = pk2<kBf16>(__uint_as_float(o[8 * c + 0]) * inv, __uint_as_float(o[8 * c + 1]) * inv);
        v.y = pk2<kBf16>(__uint_as_float(o[8 * c + 2]) * inv, __uint_as_float(o[8 * c + 3]) * inv);
        v.z = pk2<kBf16>(__uint_as_float(o[8 * c + 4]) * inv, __uint_as_float(o[8 * c + 5]) * inv);
        v.w = pk2<kBf16>(__uint_as_float(o[8 * c + 6]) * inv, __uint_as_float(o[8 * c + 7]) * inv);
        *reinterpret_cast<uint4*>(sO + sw(r, c)) = v;
      }
      fence_proxy_async_smem();
      named_bar_sync(1, 128);
      if (storer) {
        tma_store_2d(&map_ctx, sO, h * 64, req * S + qb * 128);
        tma_store_commit();
      }
    }
    if (storer) tma_store_wait_all<0>();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

}  // namespace

void launch_attention_tc(const AttnPlan& p, const int* lens, int n_req, int heads, int causal,
                         cudaStream_t stream) {
  if (n_req <= 0) return;
  const float scale_log2 = 1.4426950408889634f / sqrtf(64.0f);
  const int items = n_req * heads;
  const int grid = items < device_sm_count() ? items : device_sm_count();
  static bool configured[2] = {false, false};
  const int bf = p.precision == 1 ? 1 : 0;
  if (!configured[bf]) {
    if (bf) {
      HMI_CUDA(cudaFuncSetAttribute(attention_tc_kernel<true>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
    } else {
      HMI_CUDA(cudaFuncSetAttribute(attention_tc_kernel<false>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
    }
    configured[bf] = true;
  }
  if (bf) {
    launch_pdl(attention_tc_kernel<true>, dim3(grid), dim3(kTcThreads), kSmem, stream, p.map_qkv,
               p.map_ctx, lens, items, heads, p.d, causal, scale_log2);
  } else {
    launch_pdl(attention_tc_kernel<false>, dim3(grid), dim3(kTcThreads), kSmem, stream, p.map_qkv,
               p.map_ctx, lens, items, heads, p.d, causal, scale_log2);
  }
  HMI_CUDA(cudaGetLastError());
}

bool attention_long_tc_ok(int S) { return S % 128 == 0 && S >= 256 && S <= 128 * kLMaxBlocks; }

void launch_attention_long_tc(const AttnPlan& p, const int* lens, int n_req, int S, int heads,
                              int causal, cudaStream_t stream) {
  if (n_req <= 0) return;
  HMI_CHECK(attention_long_tc_ok(S) && p.d == heads * 64, HMI_CONFIG_ERROR,
            "attention: tcgen05 long path needs 256 <= S <= 512, S % 128 == 0, 64-wide heads");
  const float scale_log2 = 1.4426950408889634f / sqrtf(64.0f);
  const int nb = S / 128;
  const int items = n_req * heads * nb;
  const int grid = items < device_sm_count() ? items : device_sm_count();
  static bool configured[2] = {false, false};
  const int bf = p.precision == 1 ? 1 : 0;
  if (!configured[bf]) {
    if (bf) {
      HMI_CUDA(cudaFuncSetAttribute(attention_long_kernel<true>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, kLSmem));
    } else {
      HMI_CUDA(cudaFuncSetAttribute(attention_long_kernel<false>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, kLSmem));
    }
    configured[bf] = true;
  }
  if (bf) {
    launch_pdl(attention_long_kernel<true>, dim3(grid), dim3(kLThreads), kLSmem, stream, p.map_qkv,
               p.map_ctx, lens, items, heads, nb, p.d, causal, scale_log2);
  } else {
    launch_pdl(attention_long_kernel<false>, dim3(grid), dim3(kLThreads), kLSmem, stream,
               p.map_qkv, p.map_ctx, lens, items, heads, nb, p.d, causal, scale_log2);
  }
  HMI_CUDA(cudaGetLastError());
}

}  // namespace hmi_b200
