// SPDX-License-Identifier: Apache-2.0
//
// K1d — decode-step GEMMs (M = one generated row per request, 128 / 256 rows) as K-split
// thread-block clusters reduced through distributed shared memory.
//
//   C[M x N] = epilogue( A[M x K] . B^T )  the same operands, maps and epilogues as K1
//                                          (gemm_tcgen05.cuh), for the decode step's
//                                          QKV / O / FFN1 / FFN2 (model.cpp:35-37, :75, :79-81
//                                          run on the single new row of every request)
//
// At M = 256 the persistent K1 kernel has only 2 x N / BN tiles (24-72 CTAs), each
// streaming K x (128 + BN) x 2 bytes through one SM's TMA queue: the decode GEMMs ran at a
// few % of HBM, bound by per-SM ingress and pipeline fill, not by bytes. Here a tile's K
// range is cut across the ks CTAs of one cluster (grid = tiles x ks, ~148 CTAs):
//   warp 0      : TMA producer — all of this CTA's K blocks in flight at once (one stage
//                 per K block, no ring reuse); the weight (B) boxes are issued before
//                 griddepcontrol.wait, so they stream under the previous kernel's tail
//   warp 1      : TMEM allocator + MMA issuer (lane 0), one 128 x BN fp32 accumulator
//   warps 2..5  : drain the partial accumulator into this CTA's shared memory (over the
//                 consumed operand stages)
//   all warps   : after a cluster barrier, CTA r sums rows [r.128/ks, (r+1).128/ks) of the
//                 tile over the ks partials (DSMEM loads, fixed rank order: deterministic and
//                 independent of scheduling), applies bias / residual / ReLU and stores
//                 16-bit or f32 rows with coalesced 8- / 16-byte stores.
#include <cstdio>
#include <cstdlib>

#include "gemm_tcgen05.cuh"

namespace hmi_b200 {

namespace {

constexpr int kDecThreads = 192;
constexpr int kDecMaxKs = 8;  // portable cluster size
constexpr int kDecSmemCap = 227 * 1024;
constexpr int kDecMaxStages = 16;  // one operand stage (and barrier pair) per K block

template <int BN>
struct DecSmem {
  static constexpr int kStageBytes = kBlockM * kBlockK * 2 + BN * kBlockK * 2;
  static constexpr int kRedLd = BN + 4;  // floats per partial row (+4: conflict-free float4 rows)
  static constexpr int kRedBytes = kBlockM * kRedLd * 4;
  __device__ static int operand_bytes(int kb) { return kb * kStageBytes; }
};

__device__ __forceinline__ float4 ld_cluster_f32x4(uint32_t cluster_addr) {
  float4 v;
  // not volatile / no memory clobber: ordered after the cluster barrier by the barrier's own
  // asm (volatile, memory clobber), free to batch with each other
  asm("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
      : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
      : "r"(cluster_addr));
  return v;
}

template <bool kBf16>
__device__ __forceinline__ float2 unpack_16x2(uint32_t w) {
  if constexpr (kBf16) {
    return __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w));
  } else {
    return __half22float2(*reinterpret_cast<const __half2*>(&w));
  }
}

template <int BN, int EPI>
__global__ void __launch_bounds__(kDecThreads, 1)
    gemm_dec_kernel(const __grid_constant__ DecGemmMaps maps, const DecGemmArgs args) {
  using L = DecSmem<BN>;
  constexpr bool kBf16 = (EPI & kEpiBf16) != 0;
  constexpr bool kOutF32 = (EPI & kEpiOutF32) != 0;
  constexpr uint32_t kTmemCols = BN < 32 ? 32 : BN;
  const int ks = args.ks;
  const int nkb = args.kb_per_cta;
  const uint32_t rank = cluster_ctarank();
  const int tile = static_cast<int>(blockIdx.x) / ks;
  const int mt = tile / args.num_n_tiles;
  const int nt = tile - mt * args.num_n_tiles;
  const int kb0 = static_cast<int>(rank) * nkb;

  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + ((1024 - (raw_addr & 1023)) & 1023);
  const int body = L::operand_bytes(nkb) > L::kRedBytes ? L::operand_bytes(nkb) : L::kRedBytes;
  uint8_t* sA = smem;                                     // nkb x 16 KB
  uint8_t* sB = smem + nkb * kBlockM * kBlockK * 2;       // nkb x BN x 128 B
  float* red = reinterpret_cast<float*>(smem);            // over the operands, after the MMAs
  uint64_t* full_a = reinterpret_cast<uint64_t*>(smem + body);
  uint64_t* full_b = full_a + kDecMaxStages;
  uint64_t* tfull = full_b + kDecMaxStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&maps.a);
    tma_prefetch_desc(&maps.b);
    for (int s = 0; s < nkb; ++s) {
      mbar_init(&full_a[s], 1);
      mbar_init(&full_b[s], 1);
    }
    mbar_init(tfull, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_trigger();

  if (warp == 0) {
    if (lane == 0) {
      // weights do not depend on the previous kernel: stream them before the dependency wait
      const uint64_t pol_b = policy_evict_first();
      for (int s = 0; s < nkb; ++s) {
        mbar_arrive_expect_tx(&full_b[s], BN * kBlockK * 2);
        tma_load_3d_hint(sB + s * BN * kBlockK * 2, &maps.b, &full_b[s], (kb0 + s) * kBlockK,
                         nt * BN, 0, pol_b);
      }
      pdl_wait();
      const uint64_t pol_a = policy_evict_last();  // A rows are re-read by every N tile
      for (int s = 0; s < nkb; ++s) {
        mbar_arrive_expect_tx(&full_a[s], kBlockM * kBlockK * 2);
        tma_load_2d_hint(sA + s * kBlockM * kBlockK * 2, &maps.a, &full_a[s],
                         (kb0 + s) * kBlockK, mt * kBlockM, pol_a);
      }
    }
  } else if (warp == 1) {
    pdl_wait();
    if (lane == 0) {
      for (int s = 0; s < nkb; ++s) {
        mbar_wait(&full_b[s], 0);
        mbar_wait(&full_a[s], 0);
        tc_fence_after();
        const uint64_t a_desc = sdesc_k_sw128(smem_u32(sA + s * kBlockM * kBlockK * 2));
        const uint64_t b_desc = sdesc_k_sw128(smem_u32(sB + s * BN * kBlockK * 2));
#pragma unroll
        for (int k = 0; k < kBlockK / 16; ++k) {
          umma_f16(tmem_base, a_desc + 2 * k, b_desc + 2 * k, args.idesc, (s | k) != 0);
        }
      }
      umma_commit(tfull);
    }
  } else {
    // partial accumulator -> this CTA's shared memory (row-major, kRedLd floats per row)
    pdl_wait();
    const uint32_t q = warp & 3;  // TMEM lane quarter this warp may access
    const int row = static_cast<int>(q) * 32 + static_cast<int>(lane);
    mbar_wait(tfull, 0);
    tc_fence_after();
    float* dst = red + row * L::kRedLd;
#pragma unroll
    for (int c = 0; c < BN; c += 32) {
      uint32_t r[32];
      tmem_ld_32x32b_x32(tmem_base + ((q * 32) << 16) + c, r);
      tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 32; i += 4) {
        *reinterpret_cast<float4*>(dst + c + i) =
            make_float4(__uint_as_float(r[i]), __uint_as_float(r[i + 1]),
                        __uint_as_float(r[i + 2]), __uint_as_float(r[i + 3]));
      }
    }
    tc_fence_before();
  }
  pdl_wait();      // every thread: the reduction reads res0 and writes C
  cluster_sync();  // every partial of the tile is in its CTA's shared memory

  // ---- reduction + epilogue over this CTA's share of the tile's rows
  const int rows_per = (kBlockM + ks - 1) / ks;
  const int r0 = static_cast<int>(rank) * rows_per;
  const int r1 = min(kBlockM, r0 + rows_per);
  constexpr int kC4 = BN / 4;
  const uint32_t red_addr = smem_u32(red);
  const int col_base = nt * BN;
  for (int idx = static_cast<int>(threadIdx.x); idx < (r1 - r0) * kC4; idx += kDecThreads) {
    const int lr = r0 + idx / kC4;
    const int c = (idx - (idx / kC4) * kC4) * 4;
    const uint32_t a = red_addr + static_cast<uint32_t>((lr * L::kRedLd + c) * 4);
    float4 p[kDecMaxKs];  // every partial's load in flight before the first add
#pragma unroll
    for (int s = 0; s < kDecMaxKs; ++s) {
      if (s < ks) p[s] = ld_cluster_f32x4(mapa_shared(a, static_cast<uint32_t>(s)));
    }
    float4 v = p[0];
#pragma unroll
    for (int s = 1; s < kDecMaxKs; ++s) {  // fixed rank order
      if (s < ks) { v.x += p[s].x; v.y += p[s].y; v.z += p[s].z; v.w += p[s].w; }
    }
    const int grow = mt * kBlockM + lr;
    const int gcol = col_base + c;
    const float4 b4 = __ldg(reinterpret_cast<const float4*>(args.bias + gcol));
    v.x += b4.x; v.y += b4.y; v.z += b4.z; v.w += b4.w;
    if constexpr ((EPI & kEpiRes1) != 0) {
      const uint2 u = __ldg(reinterpret_cast<const uint2*>(
          reinterpret_cast<const uint16_t*>(args.res0) + static_cast<long long>(grow) * args.res_ld + gcol));
      const float2 f0 = unpack_16x2<kBf16>(u.x), f1 = unpack_16x2<kBf16>(u.y);
      v.x += f0.x; v.y += f0.y; v.z += f1.x; v.w += f1.y;
    }
    if constexpr ((EPI & kEpiRelu) != 0) {
      v.x = fmaxf(v.x, 0.f); v.y = fmaxf(v.y, 0.f); v.z = fmaxf(v.z, 0.f); v.w = fmaxf(v.w, 0.f);
    }
    if constexpr (kOutF32) {
      *reinterpret_cast<float4*>(reinterpret_cast<float*>(args.c) +
                                 static_cast<long long>(grow) * args.c_ld + gcol) = v;
    } else {
      *reinterpret_cast<uint2*>(reinterpret_cast<uint16_t*>(args.c) +
                                static_cast<long long>(grow) * args.c_ld + gcol) =
          make_uint2(pack_16x2<kBf16>(v.x, v.y), pack_16x2<kBf16>(v.z, v.w));
    }
  }
  cluster_sync();  // no CTA leaves while a peer may still read its partial
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<kTmemCols>(tmem_base);
  }
}

using DecFn = void (*)(DecGemmMaps, DecGemmArgs);

template <int BN, int T>
DecFn dec_pick_epi(int epi) {
  switch (epi) {
    case 0: return &gemm_dec_kernel<BN, T>;
    case kEpiRelu: return &gemm_dec_kernel<BN, T | kEpiRelu>;
    case kEpiOutF32: return &gemm_dec_kernel<BN, T | kEpiOutF32>;
    case kEpiRes1 | kEpiOutF32: return &gemm_dec_kernel<BN, T | kEpiRes1 | kEpiOutF32>;
    default: return nullptr;
  }
}

template <int BN>
DecFn dec_pick(int epi) {
  return (epi & kEpiBf16) ? dec_pick_epi<BN, kEpiBf16>(epi & ~kEpiBf16) : dec_pick_epi<BN, 0>(epi);
}

int dec_stage_bytes(int bn) { return kBlockM * kBlockK * 2 + bn * kBlockK * 2; }
int dec_red_bytes(int bn) { return kBlockM * (bn + 4) * 4; }
int dec_smem(int bn, int kb) {
  const int ops = kb * dec_stage_bytes(bn);
  return 1024 /*align*/ + (ops > dec_red_bytes(bn) ? ops : dec_red_bytes(bn)) + 512 /*barriers*/;
}

}  // namespace

// Tile width and K split: modelled per-SM time = the bytes each SM must take in
// (operand boxes of its CTAs, plus the DSMEM reads of the reduction) + a fixed cost per
// resident wave (launch, barrier setup, first-load latency); the co-resident clusters of a
// candidate come from the occupancy API (GPCs need not divide into clusters of ks).
DecGemmCfg pick_dec_cfg(int N, int K, int m_tiles, int sms, int epi) {
  DecGemmCfg best{0, 0};
  double best_cost = 1e30;
  const int nkb = K / kBlockK;
  for (int bn : {128, 64, 256}) {
    if (N % bn) continue;
    for (int ks = 1; ks <= kDecMaxKs; ++ks) {
      if (nkb % ks) continue;
      const int kb = nkb / ks;
      const int smem = dec_smem(bn, kb);
      if (smem > kDecSmemCap || kb > kDecMaxStages) continue;
      DecFn fn = bn == 64 ? dec_pick<64>(epi) : bn == 128 ? dec_pick<128>(epi) : dec_pick<256>(epi);
      if (!fn) continue;
      // the opt-in ceiling for every instantiation (one kernel serves plans of several K
      // splits; the launch's own dynamic size sets occupancy)
      HMI_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kDecSmemCap));
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(ks * (sms / ks));
      cfg.blockDim = dim3(kDecThreads);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = ks;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      int clusters = 0;
      if (cudaOccupancyMaxActiveClusters(&clusters, fn, &cfg) != cudaSuccess || clusters <= 0) {
        cudaGetLastError();
        continue;
      }
      const long ctas = static_cast<long>(N / bn) * m_tiles * ks;
      const long cap = static_cast<long>(clusters) * ks;  // co-resident CTAs
      const long waves = (ctas + cap - 1) / cap;
      long need = (ctas + sms - 1) / sms;  // CTAs sharing one SM's ingress
      if (need < waves) need = waves;
      const double in = kb * dec_stage_bytes(bn) + (ks > 1 ? dec_red_bytes(bn) * (ks - 1.0) / ks : 0.0);
      const double cost = need * in + waves * 48.0 * 1024;
      if (cost < best_cost - 1.0) {
        best_cost = cost;
        best = {bn, ks};
      }
    }
  }
  return best;
}

DecGemmPlan make_dec_gemm_plan(const GemmSpec& s, int m_tiles, DecGemmCfg force) {
  HMI_CHECK(s.K % kBlockK == 0 && s.a_rows % kBlockM == 0 && s.groups == 1 && !s.tile_slot,
            HMI_CONFIG_ERROR, "decode gemm: K % 64, rows % 128, shared weights");
  HMI_CHECK((s.epi & ~(kEpiRelu | kEpiRes1 | kEpiOutF32)) == 0 &&
                (!(s.epi & kEpiRes1) || (s.res0 && (s.epi & kEpiOutF32))),
            HMI_CONFIG_ERROR, "decode gemm: unsupported epilogue");
  DecGemmPlan p;
  if (force.bn > 0) {
    p.cfg = force;
  } else {
    p.cfg = pick_dec_cfg(s.N, s.K, m_tiles, device_sm_count(), s.epi | (s.precision == 1 ? kEpiBf16 : 0));
  }
  const int nkb = s.K / kBlockK;
  HMI_CHECK(p.cfg.bn > 0 && s.N % p.cfg.bn == 0 && dec_smem(p.cfg.bn, nkb / p.cfg.ks) <= kDecSmemCap && p.cfg.ks >= 1 && p.cfg.ks <= kDecMaxKs &&
                nkb % p.cfg.ks == 0 && nkb / p.cfg.ks <= kDecMaxStages,
            HMI_CONFIG_ERROR, "decode gemm: no tile / split fits");
  const int epi = s.epi | (s.precision == 1 ? kEpiBf16 : 0);
  DecFn fn = p.cfg.bn == 64 ? dec_pick<64>(epi) : p.cfg.bn == 128 ? dec_pick<128>(epi)
           : p.cfg.bn == 256 ? dec_pick<256>(epi) : nullptr;
  HMI_CHECK(fn != nullptr, HMI_CONFIG_ERROR, "decode gemm: unsupported tile / epilogue");
  p.fn = reinterpret_cast<void*>(fn);
  p.smem_bytes = dec_smem(p.cfg.bn, nkb / p.cfg.ks);
  HMI_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kDecSmemCap));
  const CUtensorMapDataType t16 =
      s.precision == 1 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  p.maps.a = make_tmap_2d(s.a, t16, s.K, s.a_rows, s.a_ld * 2ull, kBlockK, kBlockM,
                          CU_TENSOR_MAP_SWIZZLE_128B);
  p.maps.b = make_tmap_3d(s.b, t16, s.K, s.N, 1, s.b_ld * 2ull,
                          s.b_group_stride_bytes ? s.b_group_stride_bytes : size_t(s.N) * s.b_ld * 2,
                          kBlockK, p.cfg.bn, CU_TENSOR_MAP_SWIZZLE_128B);
  p.args = DecGemmArgs{};
  p.args.num_n_tiles = s.N / p.cfg.bn;
  p.args.ks = p.cfg.ks;
  p.args.kb_per_cta = nkb / p.cfg.ks;
  p.args.bias = s.bias;
  p.args.res0 = s.res0;
  p.args.res_ld = s.res_ld;
  p.args.c = s.c;
  p.args.c_ld = s.c_ld;
  p.args.idesc = idesc_f16(kBlockM, p.cfg.bn, s.precision == 1 ? 1u : 0u);
  p.max_rows = s.a_rows;
  if (std::getenv("HMI_DEBUG_PLAN")) {
    std::fprintf(stderr, "decode gemm plan: N=%d K=%d bn=%d ks=%d smem=%d\n", s.N, s.K, p.cfg.bn,
                 p.cfg.ks, p.smem_bytes);
  }
  return p;
}

void launch_dec_gemm(const DecGemmPlan& p, int M, cudaStream_t stream) {
  if (M <= 0) return;
  HMI_CHECK(M % kBlockM == 0 && M <= p.max_rows, HMI_DIMENSION_ERROR,
            "decode gemm: M must be a multiple of 128 within the planned buffer");
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((M / kBlockM) * p.args.num_n_tiles * p.cfg.ks);
  cfg.blockDim = dim3(kDecThreads);
  cfg.dynamicSmemBytes = p.smem_bytes;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = p.cfg.ks;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  HMI_CUDA(cudaLaunchKernelEx(&cfg, reinterpret_cast<DecFn>(p.fn), p.maps, p.args));
}

}  // namespace hmi_b200
