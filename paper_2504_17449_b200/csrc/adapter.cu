// SPDX-License-Identifier: Apache-2.0
//
// K2 fused: the whole per-tenant adapter of one layer in ONE persistent kernel.
//
//   mid = ReLU(a . Wd + bd)                      adapter_apply down  (proj/src/transformer/model.cpp:15-17)
//   y1  = mid . Wu + bu + a + LN2_{l-1}(y2)      up + skip (model.cpp:18-21) + residual (model.cpp:91)
//
// and the per-row partial (sum, sum of squares) of y1 for the LN1 consumers (the LayerNorm
// folding of gemm_tcgen05.cuh). Each 128-row M tile is one request, so one tenant: its HBM
// slot (tile_slot[m]) supplies Wd^T [64][d], Wu^T [d][64], bd, bu — the reference's
// per-element parameter choice of batched_adapter_apply (proj/src/adapters/stacked.cpp:44-64)
// without the stack() copy (stacked.cpp:12-42).
//
// Replaces the two grouped GEMMs (down: reads a, writes mid; up: reads mid, a, h, writes y1):
// `a` is read once from HBM (the residual re-read hits L2), mid never leaves the SM.
//
// Roles (352 threads, 1 CTA per SM, persistent over M tiles):
//   warp 0  : operand producer: per tile 12 (a, Wd) K blocks, then 6 Wu N chunks, through one
//             ring of kStages 24 KB stages (so the next tile's K blocks prefetch behind the
//             current tile's up-projection)
//   warp 1  : TMEM allocator + MMA issuer: mid acc (128 x 64) over K = d; after the epilogue
//             has written ReLU(mid) to smem, 6 x (128 x 128) y chunks over K = 64 into two
//             alternating TMEM accumulators
//   warp 2  : residual producer: (a, h) 64-column boxes of the tile into a 3-slot ring
//   warps 3-10: epilogue. E1: mid acc -> +bd, ReLU -> 16-bit, swizzled into smem (the A
//             operand of the up MMAs). E2: a + LN(h) from the residual ring (slot released
//             at once) -> + y chunk + bu -> stats -> 16-bit -> per-warp staging -> TMA store.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <cstdint>

#include "adapter.hpp"
#include "kernels.hpp"
#include "sm100.cuh"

namespace hmi_b200 {

namespace {

constexpr int kThreads = 352;
constexpr int kStages = 3;
constexpr int kStageBytes = 24576;     // A 128 x 64 (16 KB) + Wd 64 x 64 (8 KB); or Wu 128 x 64
constexpr int kResSlots = 3;
constexpr int kResBytes = 32768;       // a box + h box, 128 rows x 64 columns each
constexpr int kVecBytes = 768;         // per residual slot: the chunk's 64 bu, gamma, beta floats
constexpr int kBox = 16384;
constexpr int kUpN = 128;              // y chunk width
constexpr int kSmem = 1024 + kStages * kStageBytes + kBox /*mid*/ + kResSlots * kResBytes +
                     8 * 4096 /*staging*/ + kResSlots * kVecBytes + 256;

template <bool kBf16>
__device__ __forceinline__ float2 unpack2(uint32_t w) {
  if constexpr (kBf16) {
    return __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w));
  } else {
    return __half22float2(*reinterpret_cast<const __half2*>(&w));
  }
}

template <bool kBf16>
__device__ __forceinline__ uint32_t pack2(float a, float b) {
  if constexpr (kBf16) {
    const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<const uint32_t*>(&h);
  } else {
    const __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<const uint32_t*>(&h);
  }
}

template <bool kBf16>
__global__ void __launch_bounds__(kThreads, 1)
    adapter_fused_kernel(const __grid_constant__ AdapterMaps maps, const AdapterArgs args) {
  extern __shared__ uint8_t raw[];
  uint8_t* base = raw + ((1024 - (smem_u32(raw) & 1023)) & 1023);
  uint8_t* ring = base;
  uint8_t* midA = ring + kStages * kStageBytes;
  uint8_t* res = midA + kBox;
  uint8_t* vec = res + kResSlots * kResBytes + 8 * 4096;  // [kResSlots][kVecBytes]
  uint64_t* bar = reinterpret_cast<uint64_t*>(vec + kResSlots * kVecBytes);
  uint64_t* full = bar;                          // [kStages]
  uint64_t* empty = bar + kStages;               // [kStages]
  uint64_t* res_full = bar + 2 * kStages;        // [kResSlots]
  uint64_t* res_empty = res_full + kResSlots;    // [kResSlots]
  uint64_t* macc_full = res_empty + kResSlots;   // mid accumulator complete
  uint64_t* macc_empty = macc_full + 1;          // mid accumulator drained (8 warps)
  uint64_t* mid_full = macc_full + 2;            // ReLU(mid) written to smem (8 warps)
  uint64_t* yacc_full = macc_full + 3;           // [2]
  uint64_t* yacc_empty = macc_full + 5;          // [2] (8 warps)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(macc_full + 7);
  // residual chunk index currently owned by each ring slot. The two column halves consume
  // alternate chunks, so a half can run a full ring lap ahead of the other; with an odd slot
  // count a parity wait alone could then pass on the slot's previous fill. A consumer first
  // waits for the producer to tag the slot with its chunk, then on the (now unambiguous) phase.
  volatile uint32_t* res_tag = tmem_slot + 1;  // [kResSlots]

  const uint32_t warp = warp_id(), lane = lane_id();
  const int d = args.d;
  const int n_kb = d / 64;
  const int n_up = d / kUpN;
  const int n_res = d / 64;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&maps.a);
    tma_prefetch_desc(&maps.h);
    tma_prefetch_desc(&maps.wd);
    tma_prefetch_desc(&maps.wu);
    tma_prefetch_desc(&maps.out);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < kResSlots; ++s) {
      mbar_init(&res_full[s], 1);
      mbar_init(&res_empty[s], 4);
      res_tag[s] = 0xffffffffu;
    }
    mbar_init(macc_full, 1);
    mbar_init(macc_empty, 8);
    mbar_init(mid_full, 8);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&yacc_full[s], 1);
      mbar_init(&yacc_empty[s], 8);
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
  if (args.ready != nullptr) {
    // fine pipeline: wait on the device for this layer's adapter copies (the copy stream
    // writes the batch's sequence number after them) instead of a stream-level event wait,
    // which would cut the programmatic-launch chain O-proj -> adapter
    if (threadIdx.x == 0) {
      const uint64_t t0 = globaltimer_ns();
      while (ld_acquire_gpu(args.ready) - args.ready_seq > 0x7fffffffu) {  // wrap-safe <
        if (globaltimer_ns() - t0 > 20ull * 1000 * 1000 * 1000) {  // 20 s: never, unless broken
          atomicExch(args.err, HMI_SCHEDULING_BUG);
          break;
        }
        __nanosleep(256);
      }
      fence_proxy_async_global();
    }
    __syncthreads();
  }
  // TMEM columns: mid acc 0..63, y acc[0] 128..255, y acc[1] 256..383

  if (warp == 0) {
    // ------------------------------------------------------------ operand producer
    if (lane == 0) {
      const uint64_t pol_once = policy_evict_first();  // tenant weights
      uint32_t stage = 0, phase = 0;
      for (int mt = blockIdx.x; mt < args.num_m_tiles; mt += gridDim.x) {
        const int grp = __ldg(&args.tile_slot[mt]);
        for (int kb = 0; kb < n_kb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* st = ring + stage * kStageBytes;
          mbar_arrive_expect_tx(&full[stage], kBox + 8192);
          tma_load_2d(st, &maps.a, &full[stage], kb * 64, mt * 128);
          tma_load_3d_hint(st + kBox, &maps.wd, &full[stage], kb * 64, 0, grp, pol_once);
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
        for (int c = 0; c < n_up; ++c) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* st = ring + stage * kStageBytes;
          mbar_arrive_expect_tx(&full[stage], kBox);
          tma_load_3d_hint(st, &maps.wu, &full[stage], 0, c * kUpN, grp, pol_once);
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 2) {
    // ------------------------------------------------------------ residual producer
    if (lane == 0) {
      const uint64_t pol_once = policy_evict_first();
      uint32_t slot = 0, phase = 0, jg = 0;
      for (int mt = blockIdx.x; mt < args.num_m_tiles; mt += gridDim.x) {
        const long long grp = __ldg(&args.tile_slot[mt]);
        for (int j = 0; j < n_res; ++j, ++jg) {
          mbar_wait(&res_empty[slot], phase ^ 1);
          res_tag[slot] = jg;
          uint8_t* rs = res + slot * kResBytes;
          const bool ln = args.r_stats != nullptr;
          mbar_arrive_expect_tx(&res_full[slot], 2 * kBox + (ln ? 768 : 256));
          tma_load_2d_hint(rs, &maps.a, &res_full[slot], j * 64, mt * 128, pol_once);
          tma_load_2d_hint(rs + kBox, &maps.h, &res_full[slot], j * 64, mt * 128, pol_once);
          uint8_t* vs = vec + slot * kVecBytes;
          bulk_load(vs, args.bu + grp * args.slot_floats + j * 64, 256, &res_full[slot]);
          if (ln) {
            bulk_load(vs + 256, args.r_gamma + j * 64, 256, &res_full[slot]);
            bulk_load(vs + 512, args.r_beta + j * 64, 256, &res_full[slot]);
          }
          if (++slot == kResSlots) { slot = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      const uint32_t id_d = idesc_f16(128, 64, kBf16 ? 1u : 0u);
      const uint32_t id_u = idesc_f16(128, kUpN, kBf16 ? 1u : 0u);
      uint32_t stage = 0, phase = 0, tile_ph = 0, u = 0;
      for (int mt = blockIdx.x; mt < args.num_m_tiles; mt += gridDim.x) {
        mbar_wait(macc_empty, tile_ph ^ 1);
        tc_fence_after();
        for (int kb = 0; kb < n_kb; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t st = smem_u32(ring + stage * kStageBytes);
          const uint64_t ad = sdesc_k_sw128(st);
          const uint64_t bd = sdesc_k_sw128(st + kBox);
#pragma unroll
          for (int k = 0; k < 4; ++k) umma_f16(tmem, ad + 2 * k, bd + 2 * k, id_d, (kb | k) != 0);
          umma_commit(&empty[stage]);
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
        umma_commit(macc_full);
        mbar_wait(mid_full, tile_ph);
        tc_fence_after();
        const uint64_t md = sdesc_k_sw128(smem_u32(midA));
        for (int c = 0; c < n_up; ++c, ++u) {
          const uint32_t b = u & 1;
          mbar_wait(&yacc_empty[b], ((u >> 1) & 1) ^ 1);
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint64_t wd = sdesc_k_sw128(smem_u32(ring + stage * kStageBytes));
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            umma_f16(tmem + 128 + b * kUpN, md + 2 * k, wd + 2 * k, id_u, k != 0);
          }
          umma_commit(&empty[stage]);
          umma_commit(&yacc_full[b]);
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
        tile_ph ^= 1;
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue (8 warps)
    const uint32_t q = warp & 3;                       // TMEM lane quarter
    const int half = static_cast<int>(warp - 3) >> 2;  // column half of every chunk
    const int r = static_cast<int>(q * 32 + lane);     // tile row owned by this thread
    const uint32_t lane_off = (q * 32) << 16;
    uint32_t tile_ph = 0, u = 0, tile_j0 = 0;
    uint8_t* stg = res + kResSlots * kResBytes + (warp - 3) * 4096;  // output staging
    for (int mt = blockIdx.x; mt < args.num_m_tiles; mt += gridDim.x) {
      const int grp = __ldg(&args.tile_slot[mt]);
      const int row = mt * 128 + r;
      float2 rst = make_float2(0.f, 1.f);
      if (args.r_stats != nullptr) {  // LN2 of the previous layer, applied to h on the fly
        const float4* p = reinterpret_cast<const float4*>(args.r_stats +
                                                          static_cast<long long>(row) * args.r_stats_ld);
        float4 q[8];  // r_stats_ld = 16 float2: every partial in one round trip
#pragma unroll
        for (int i = 0; i < 8; ++i)
          q[i] = 2 * i < args.r_stats_n ? __ldg(p + i) : make_float4(0.f, 0.f, 0.f, 0.f);
        float s1 = 0.f, s2 = 0.f;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          s1 += q[i].x;
          s2 += q[i].y;
          if (2 * i + 1 < args.r_stats_n) {
            s1 += q[i].z;
            s2 += q[i].w;
          }
        }
        const float mean = s1 * args.inv_n;
        const float var = fmaxf(s2 * args.inv_n - mean * mean, 0.0f);
        rst = make_float2(mean, 1.0f / sqrtf(var + 1e-5f));
      }
      // ---- E1: mid = ReLU(acc + bd) -> 16-bit A operand (columns half*32 .. +32)
      {
        const float* bdp = args.bd + static_cast<long long>(grp) * args.slot_floats + half * 32;
        mbar_wait(macc_full, tile_ph);
        tc_fence_after();
        uint32_t t[32];
        tmem_ld_32x32b_x32(tmem + lane_off + half * 32, t);
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(macc_empty);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          float v[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            v[e] = fmaxf(__uint_as_float(t[8 * c + e]) + __ldg(bdp + 8 * c + e), 0.0f);
          }
          const int chunk = half * 4 + c;
          *reinterpret_cast<uint4*>(midA + r * 128 + ((chunk ^ (r & 7)) << 4)) =
              make_uint4(pack2<kBf16>(v[0], v[1]), pack2<kBf16>(v[2], v[3]),
                         pack2<kBf16>(v[4], v[5]), pack2<kBf16>(v[6], v[7]));
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(mid_full);
      }
      // ---- E2: y chunks. Residual chunk j = 2c + half of this tile lives in ring slot
      // (tile_j0 + j) % kResSlots; it is released as soon as bu + a + LN(h) is in registers.
      float s1 = 0.f, s2 = 0.f;
      for (int c = 0; c < n_up; ++c, ++u) {
        const uint32_t b = u & 1;
        const int col0 = c * kUpN + half * 64;
        const uint32_t j = tile_j0 + 2 * c + half;
        const uint32_t slot = j % kResSlots;
        const uint8_t* rs = res + slot * kResBytes;
        const float* s_bu = reinterpret_cast<const float*>(vec + slot * kVecBytes);
        const float* s_g = s_bu + 64;
        const float* s_b = s_bu + 128;
        float v[64];
        if (lane == 0) {
          while (res_tag[slot] != j) {
          }
        }
        __syncwarp();
        mbar_wait(&res_full[slot], (j / kResSlots) & 1);
#pragma unroll
        for (int k = 0; k < 8; ++k) {  // a (skip) + LN(h) or h (residual)
          const int off = r * 128 + ((k ^ (r & 7)) << 4);
          const uint4 ua = *reinterpret_cast<const uint4*>(rs + off);
          const uint4 uh = *reinterpret_cast<const uint4*>(rs + kBox + off);
          const uint32_t wa[4] = {ua.x, ua.y, ua.z, ua.w};
          const uint32_t wh[4] = {uh.x, uh.y, uh.z, uh.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int i = 8 * k + 2 * e;
            const float2 fa = unpack2<kBf16>(wa[e]);
            const float2 fh = unpack2<kBf16>(wh[e]);
            const float2 bu2 = *reinterpret_cast<const float2*>(s_bu + i);
            if (args.r_stats != nullptr) {
              const float2 g = *reinterpret_cast<const float2*>(s_g + i);
              const float2 be = *reinterpret_cast<const float2*>(s_b + i);
              v[i] = bu2.x + fa.x + ((fh.x - rst.x) * rst.y * g.x + be.x);
              v[i + 1] = bu2.y + fa.y + ((fh.y - rst.x) * rst.y * g.y + be.y);
            } else {
              v[i] = bu2.x + fa.x + fh.x;
              v[i + 1] = bu2.y + fa.y + fh.y;
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&res_empty[slot]);
        mbar_wait(&yacc_full[b], (u >> 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          uint32_t t[32];
          tmem_ld_32x32b_x32(tmem + lane_off + 128 + b * kUpN + half * 64 + 32 * hh, t);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) v[32 * hh + i] += __uint_as_float(t[i]);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&yacc_empty[b]);
#pragma unroll
        for (int i = 0; i < 64; ++i) {
          s1 += v[i];
          s2 += v[i] * v[i];
        }
        // this warp's 32 x 64 output box -> its own staging buffer -> TMA store
        if (lane == 0) tma_store_wait_read<0>();
        __syncwarp();
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          *reinterpret_cast<uint4*>(stg + lane * 128 + ((k ^ (lane & 7)) << 4)) =
              make_uint4(pack2<kBf16>(v[8 * k], v[8 * k + 1]), pack2<kBf16>(v[8 * k + 2], v[8 * k + 3]),
                         pack2<kBf16>(v[8 * k + 4], v[8 * k + 5]),
                         pack2<kBf16>(v[8 * k + 6], v[8 * k + 7]));
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          tma_store_2d(&maps.out, stg, col0, mt * 128 + static_cast<int>(q) * 32);
          tma_store_commit();
        }
      }
      tile_j0 += n_res;
      if (row < args.M) {
        args.stats_out[static_cast<long long>(row) * args.stats_ld + half] = make_float2(s1, s2);
      }
      tile_ph ^= 1;
    }
    if (lane == 0) tma_store_wait_all<0>();
    __syncwarp();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

}  // namespace

AdapterPlan make_adapter_plan(const AdapterSpec& s) {
  HMI_CHECK(s.r_pad == 64, HMI_CONFIG_ERROR, "fused adapter: bottleneck must pad to 64");
  HMI_CHECK(s.d % kUpN == 0 && s.d >= kUpN, HMI_CONFIG_ERROR,
            "fused adapter: hidden size must be a multiple of 128");
  HMI_CHECK(s.rows % 128 == 0, HMI_CONFIG_ERROR, "fused adapter: rows must be a multiple of 128");
  HMI_CHECK(s.r_stats == nullptr || (s.stats_ld == 16 && s.r_stats_n <= 16), HMI_CONFIG_ERROR,
            "fused adapter: statistics rows of 16 float2");
  auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  HMI_CHECK(al16(s.arena + s.off_bu) && s.slot_bytes % 16 == 0 &&
                (s.r_stats == nullptr || (al16(s.r_gamma) && al16(s.r_beta))),
            HMI_CONFIG_ERROR, "fused adapter: bias / LayerNorm vectors must be 16-byte aligned");
  const CUtensorMapDataType t16 =
      s.precision == 1 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  AdapterPlan p;
  p.maps.a = make_tmap_2d(s.a, t16, s.d, s.rows, s.d * 2ull, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B);
  p.maps.h = make_tmap_2d(s.h, t16, s.d, s.rows, s.d * 2ull, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B);
  p.maps.out = make_tmap_2d(s.out, t16, s.d, s.rows, s.d * 2ull, 64, 32, CU_TENSOR_MAP_SWIZZLE_128B);
  p.maps.wd = make_tmap_3d(s.arena, t16, s.d, s.r_pad, s.n_slots, s.d * 2ull, s.slot_bytes, 64, 64,
                           CU_TENSOR_MAP_SWIZZLE_128B);
  p.maps.wu = make_tmap_3d(s.arena + s.off_wu, t16, s.r_pad, s.d, s.n_slots, s.r_pad * 2ull,
                           s.slot_bytes, 64, kUpN, CU_TENSOR_MAP_SWIZZLE_128B);
  AdapterArgs& a = p.args;
  a.d = s.d;
  a.tile_slot = s.tile_slot;
  a.bd = reinterpret_cast<const float*>(s.arena + s.off_bd);
  a.bu = reinterpret_cast<const float*>(s.arena + s.off_bu);
  a.slot_floats = static_cast<long long>(s.slot_bytes / 4);
  a.stats_out = s.stats_out;
  a.stats_ld = s.stats_ld;
  a.r_stats = s.r_stats;
  a.r_stats_n = s.r_stats_n;
  a.r_stats_ld = s.stats_ld;
  a.r_gamma = s.r_gamma;
  a.r_beta = s.r_beta;
  a.inv_n = 1.0f / static_cast<float>(s.d);
  p.precision = s.precision;
  p.max_rows = s.rows;
  return p;
}

void launch_adapter(const AdapterPlan& p, int rows, cudaStream_t stream, const uint32_t* ready,
                    uint32_t ready_seq, int32_t* err) {
  if (rows <= 0) return;
  HMI_CHECK(rows % 128 == 0 && rows <= p.max_rows, HMI_DIMENSION_ERROR,
            "fused adapter: rows must be a multiple of 128 within the plan");
  static bool configured[2] = {false, false};
  const int bf = p.precision == 1 ? 1 : 0;
  if (!configured[bf]) {
    if (bf) {
      HMI_CUDA(cudaFuncSetAttribute(adapter_fused_kernel<true>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
    } else {
      HMI_CUDA(cudaFuncSetAttribute(adapter_fused_kernel<false>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
    }
    configured[bf] = true;
  }
  AdapterArgs a = p.args;
  a.ready = ready;
  a.ready_seq = ready_seq;
  a.err = err;
  a.M = rows;
  a.num_m_tiles = rows / 128;
  const int grid = a.num_m_tiles < device_sm_count() ? a.num_m_tiles : device_sm_count();
  if (bf) {
    launch_pdl(adapter_fused_kernel<true>, dim3(grid), dim3(kThreads), kSmem, stream, p.maps, a);
  } else {
    launch_pdl(adapter_fused_kernel<false>, dim3(grid), dim3(kThreads), kSmem, stream, p.maps, a);
  }
  HMI_CUDA(cudaGetLastError());
}

}  // namespace hmi_b200
