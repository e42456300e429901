// SPDX-License-Identifier: Apache-2.0
//
// Host side of K1/K2: plan construction (TMA maps encoded once per buffer
// binding), template dispatch, and the standalone probe entry point.
#include "gemm.hpp"

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "gemm_tcgen05.cuh"

namespace hmi_b200 {

namespace {

using KernelFn = void (*)(GemmMaps, GemmArgs);

template <int BN, int EPI, bool C2>
KernelFn kernel_ptr() {
  if constexpr (C2) {
    return reinterpret_cast<KernelFn>(&gemm2_tcgen05_kernel<BN, EPI>);
  } else {
    return reinterpret_cast<KernelFn>(&gemm_tcgen05_kernel<BN, EPI>);
  }
}

template <int BN, int T, bool C2>
KernelFn pick_epi_t(int epi) {
  switch (epi) {
    case 0: return kernel_ptr<BN, T, C2>();
    case kEpiRelu: return kernel_ptr<BN, T | kEpiRelu, C2>();
    case kEpiRes1: return kernel_ptr<BN, T | kEpiRes1, C2>();
    case kEpiRes2: return kernel_ptr<BN, T | kEpiRes2, C2>();
    case kEpiOutF32: return kernel_ptr<BN, T | kEpiOutF32, C2>();
    case kEpiRes1 | kEpiOutF32: return kernel_ptr<BN, T | kEpiRes1 | kEpiOutF32, C2>();
    case kEpiRes2 | kEpiOutF32: return kernel_ptr<BN, T | kEpiRes2 | kEpiOutF32, C2>();
    // LayerNorm folding
    case kEpiFoldLN: return kernel_ptr<BN, T | kEpiFoldLN, C2>();
    case kEpiRelu | kEpiFoldLN: return kernel_ptr<BN, T | kEpiRelu | kEpiFoldLN, C2>();
    case kEpiRes1 | kEpiRes0LN | kEpiStats:
      return kernel_ptr<BN, T | kEpiRes1 | kEpiRes0LN | kEpiStats, C2>();
    case kEpiRes2 | kEpiStats: return kernel_ptr<BN, T | kEpiRes2 | kEpiStats, C2>();
    case kEpiRes2 | kEpiRes1LN | kEpiStats:
      return kernel_ptr<BN, T | kEpiRes2 | kEpiRes1LN | kEpiStats, C2>();
    default: break;
  }
  if constexpr (C2) {  // O projection + tenant up projection (+ LN'd residual) + statistics
    switch (epi) {
      case kEpiExt | kEpiRes1 | kEpiStats:
        return kernel_ptr<BN, T | kEpiExt | kEpiRes1 | kEpiStats, true>();
      case kEpiExt | kEpiRes1 | kEpiRes0LN | kEpiStats:
        return kernel_ptr<BN, T | kEpiExt | kEpiRes1 | kEpiRes0LN | kEpiStats, true>();
      default: break;
    }
  }
  if constexpr (!C2 && BN <= 192) {  // adapter up with TMA-staged residuals
    switch (epi) {
      case kEpiRes2 | kEpiStats | kEpiResTma:
        return kernel_ptr<BN, T | kEpiRes2 | kEpiStats | kEpiResTma, false>();
      case kEpiRes2 | kEpiRes1LN | kEpiStats | kEpiResTma:
        return kernel_ptr<BN, T | kEpiRes2 | kEpiRes1LN | kEpiStats | kEpiResTma, false>();
      default: break;
    }
  }
  return nullptr;
}

template <int BN, bool C2>
KernelFn pick_epi(int epi) {
  return (epi & kEpiBf16) ? pick_epi_t<BN, kEpiBf16, C2>(epi & ~kEpiBf16)
                          : pick_epi_t<BN, 0, C2>(epi);
}

KernelFn pick_kernel(int bn, int epi, bool c2, int* smem_bytes) {
  if (c2) {
    switch (bn) {
      case 128:
        *smem_bytes = pair_svec(epi) ? Gemm2Smem<128, true>::kTotal : Gemm2Smem<128>::kTotal;
        return pick_epi<128, true>(epi);
      case 192:
        *smem_bytes = pair_svec(epi) ? Gemm2Smem<192, true>::kTotal : Gemm2Smem<192>::kTotal;
        return pick_epi<192, true>(epi);
      case 256:
        *smem_bytes = pair_svec(epi) ? Gemm2Smem<256, true>::kTotal : Gemm2Smem<256>::kTotal;
        return pick_epi<256, true>(epi);
      default: return nullptr;
    }
  }
  const bool rt = (epi & kEpiResTma) != 0;
#define HMI_SMEM(B) \
  (rt ? (B <= 192 ? GemmSmem<(B <= 192 ? B : 64), true>::kTotal : 0) : GemmSmem<B>::kTotal)
  switch (bn) {
    case 64: *smem_bytes = HMI_SMEM(64); return pick_epi<64, false>(epi);
    case 128: *smem_bytes = HMI_SMEM(128); return pick_epi<128, false>(epi);
    case 192: *smem_bytes = HMI_SMEM(192); return pick_epi<192, false>(epi);
    case 256: *smem_bytes = HMI_SMEM(256); return pick_epi<256, false>(epi);
    default: return nullptr;
  }
#undef HMI_SMEM
}

}  // namespace

GemmPlan make_gemm_plan(const GemmSpec& s) {
  HMI_CHECK(s.K % kBlockK == 0, HMI_CONFIG_ERROR, "gemm: K must be a multiple of 64");
  HMI_CHECK(s.bn == 64 || s.bn == 128 || s.bn == 192 || s.bn == 256, HMI_CONFIG_ERROR,
            "gemm: unsupported N tile");
  HMI_CHECK(s.N % s.bn == 0, HMI_CONFIG_ERROR, "gemm: N must be a multiple of the N tile");
  HMI_CHECK(s.a_rows % kBlockM == 0, HMI_CONFIG_ERROR, "gemm: A rows must be a multiple of 128");
  GemmPlan p;
  const int epi = s.epi | (s.precision == 1 ? kEpiBf16 : 0);
  const bool ext = (s.epi & kEpiExt) != 0;
  const bool c2 = s.cta2 && s.groups == 1 && (s.tile_slot == nullptr || ext) && s.bn >= 128;
  HMI_CHECK(!ext || (c2 && s.tile_slot && s.ext_a && s.ext_b && s.ext_bias && s.ext_k > 0 &&
                     s.ext_k % kBlockK == 0),
            HMI_CONFIG_ERROR, "gemm: tenant extension needs the pair kernel and its operands");
  p.two_cta = c2;
  p.fn = reinterpret_cast<void*>(pick_kernel(s.bn, epi, c2, &p.smem_bytes));
  HMI_CHECK(p.fn != nullptr, HMI_CONFIG_ERROR, "gemm: unsupported epilogue");
  const CUtensorMapDataType t16 =
      s.precision == 1 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  p.maps.a = make_tmap_2d(s.a, t16, s.K, s.a_rows, s.a_ld * 2ull, kBlockK, kBlockM,
                         CU_TENSOR_MAP_SWIZZLE_128B);
  p.maps.b = make_tmap_3d(s.b, t16, s.K, s.N, s.groups, s.b_ld * 2ull, s.b_group_stride_bytes,
                         kBlockK, c2 ? s.bn / 2 : s.bn, CU_TENSOR_MAP_SWIZZLE_128B);
  const bool f32 = (s.epi & kEpiOutF32) != 0;
  p.maps.c = make_tmap_2d(s.c, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : t16, s.N, s.a_rows,
                         s.c_ld * (f32 ? 4ull : 2ull), f32 ? 32 : 64, 32,
                         CU_TENSOR_MAP_SWIZZLE_128B);
  p.maps.r0 = p.maps.c;
  p.maps.r1 = p.maps.c;
  if (s.epi & kEpiResTma) {
    HMI_CHECK(s.res0 && s.res1 && !c2, HMI_CONFIG_ERROR, "gemm: TMA residuals need 2 residuals (1-CTA)");
    p.maps.r0 = make_tmap_2d(s.res0, t16, s.N, s.a_rows, s.res_ld * 2ull, 64, 128,
                             CU_TENSOR_MAP_SWIZZLE_128B);
    p.maps.r1 = make_tmap_2d(s.res1, t16, s.N, s.a_rows, s.res_ld * 2ull, 64, 128,
                             CU_TENSOR_MAP_SWIZZLE_128B);
  }
  p.precision = s.precision;
  p.bn = s.bn;
  if (c2) {
    // wave-tail sub-tile widths must stay multiples of 64 columns (the epilogue's store chunk)
    const int g = s.bn / 64;
    p.tail_s0 = g % 2 == 0 ? 2 : g % 3 == 0 ? 3 : 0;
    p.tail_s1 = g % 4 == 0 ? 4 : p.tail_s0;
    if (p.tail_s0) {
      p.maps.r0 = make_tmap_3d(s.b, t16, s.K, s.N, s.groups, s.b_ld * 2ull, s.b_group_stride_bytes,
                               kBlockK, s.bn / (2 * p.tail_s0), CU_TENSOR_MAP_SWIZZLE_128B);
      p.maps.r1 = make_tmap_3d(s.b, t16, s.K, s.N, s.groups, s.b_ld * 2ull, s.b_group_stride_bytes,
                               kBlockK, s.bn / (2 * p.tail_s1), CU_TENSOR_MAP_SWIZZLE_128B);
    }
  }
  p.maps.xa = p.maps.xb = p.maps.xb0 = p.maps.xb1 = p.maps.res = p.maps.c;
  if (c2 && (s.epi & kEpiRes1) && !(s.epi & (kEpiRes2 | kEpiOutF32))) {
    HMI_CHECK(s.res0 != nullptr, HMI_CONFIG_ERROR, "gemm: residual missing");
    p.maps.res = make_tmap_2d(s.res0, t16, s.N, s.a_rows, s.res_ld * 2ull, 64, 32,
                              CU_TENSOR_MAP_SWIZZLE_128B);
  }
  if (ext) {
    // ext rows: a_rows + 128 (the last 128 are the zero rows of the other CTA's half)
    p.maps.xa = make_tmap_2d(s.ext_a, t16, s.ext_k, s.a_rows + kBlockM, s.ext_k * 2ull, kBlockK,
                             kBlockM, CU_TENSOR_MAP_SWIZZLE_128B);
    auto xb = [&](int width) {
      return make_tmap_3d(s.ext_b, t16, s.ext_k, s.N, s.ext_groups, s.ext_b_ld * 2ull,
                          s.ext_b_stride, kBlockK, width, CU_TENSOR_MAP_SWIZZLE_128B);
    };
    p.maps.xb = xb(s.bn / 2);
    if (p.tail_s0) {
      p.maps.xb0 = xb(s.bn / (2 * p.tail_s0));
      p.maps.xb1 = xb(s.bn / (2 * p.tail_s1));
    }
  }
  p.args = GemmArgs{};
  p.args.N = s.N;
  p.args.K = s.K;
  p.args.num_n_tiles = s.N / s.bn;
  p.args.bias = s.bias;
  p.args.bias_slot_stride = s.bias_group_stride;
  p.args.tile_slot = s.tile_slot;
  p.args.res0 = reinterpret_cast<const __half*>(s.res0);
  p.args.res1 = reinterpret_cast<const __half*>(s.res1);
  p.args.res_ld = s.res_ld;
  p.args.stats_out = s.stats_out;
  p.args.stats_ld = s.stats_ld;
  p.args.a_stats = s.a_stats;
  p.args.a_stats_n = s.a_stats_n;
  p.args.colsum = s.colsum;
  p.args.r_stats = s.r_stats;
  p.args.r_stats_n = s.r_stats_n;
  p.args.r_gamma = s.r_gamma;
  p.args.r_beta = s.r_beta;
  p.args.inv_n = s.inv_n;
  if (ext) {
    p.args.ext_kb = s.ext_k / kBlockK;
    p.args.ext_zero_row = s.a_rows;
    p.args.bias2 = s.ext_bias;
    p.args.bias2_stride = s.ext_bias_stride;
  }
  if (s.epi & kEpiStats) HMI_CHECK(s.stats_out && s.stats_ld == kStatsStride && s.N % 64 == 0 && s.N / 64 <= kStatsStride, HMI_CONFIG_ERROR, "gemm: stats buffer");
  if (s.epi & kEpiFoldLN) HMI_CHECK(s.a_stats && s.colsum && s.inv_n > 0.f, HMI_CONFIG_ERROR, "gemm: fold args");
  if (s.epi & (kEpiRes0LN | kEpiRes1LN))
    HMI_CHECK(s.r_stats && s.r_gamma && s.r_beta && s.inv_n > 0.f, HMI_CONFIG_ERROR, "gemm: residual LN args");
  p.args.idesc = idesc_f16(c2 ? 2 * kBlockM : kBlockM, s.bn, s.precision == 1 ? 1u : 0u);
  p.max_rows = s.a_rows;
  if (c2) {
    // co-resident CTA pairs (GPCs need not divide evenly into clusters)
    HMI_CUDA(cudaFuncSetAttribute(p.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, p.smem_bytes));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * (device_sm_count() / 2));
    cfg.blockDim = dim3(kGemmThreads);
    cfg.dynamicSmemBytes = p.smem_bytes;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, p.fn, &cfg) != cudaSuccess || n <= 0) {
      cudaGetLastError();
      n = device_sm_count() / 2;
    }
    p.max_clusters = n;
    if (std::getenv("HMI_DEBUG_PLAN")) {
      std::fprintf(stderr, "gemm plan: pair kernel bn=%d smem=%d max_clusters=%d\n", s.bn,
                   p.smem_bytes, n);
    }
  }
  return p;
}

void launch_gemm(const GemmPlan& p, int M, cudaStream_t stream, const uint32_t* ready,
                 uint32_t ready_seq, int32_t* err) {
  if (M <= 0) return;
  HMI_CHECK(M % kBlockM == 0 && M <= p.max_rows, HMI_DIMENSION_ERROR,
            "gemm: M must be a multiple of 128 within the planned buffer");
  static std::mutex mu;
  static std::vector<void*> configured;
  {
    std::lock_guard<std::mutex> lock(mu);
    bool seen = false;
    for (void* f : configured) seen |= (f == p.fn);
    if (!seen) {
      HMI_CUDA(cudaFuncSetAttribute(p.fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    p.smem_bytes));
      configured.push_back(p.fn);
    }
  }
  GemmArgs a = p.args;
  a.M = M;
  a.num_m_tiles = M / kBlockM;
  int grid;
  a.n_main = 0;
  a.tail_split = 1;
  a.idesc_tail = a.idesc;
  a.tail_r1 = 0;
  a.ready = ready;
  a.ready_seq = ready_seq;
  a.err = err;
  HMI_CHECK(ready == nullptr || (!p.two_cta && err != nullptr), HMI_CONFIG_ERROR,
            "gemm: readiness wait needs the 1-CTA kernel and an error word");
  if (p.two_cta) {
    const int rows = 2;  // M tiles per pair unit
    const int units = (a.num_m_tiles + rows - 1) / rows * a.num_n_tiles;
    const int clusters = p.max_clusters > 0 ? p.max_clusters : device_sm_count() / rows;
    grid = rows * (units < clusters ? units : clusters);
    // the last partial wave of R units runs as R x S narrower sub-tiles (R x S <= clusters)
    const int R = units > clusters ? units % clusters : 0;
    if (p.tail_enabled && R > 0 && p.tail_s0) {
      int S = 1;
      if (p.tail_s1 > 1 && R * p.tail_s1 <= clusters) {
        S = p.tail_s1;
        a.tail_r1 = 1;
      } else if (R * p.tail_s0 <= clusters) {
        S = p.tail_s0;
      }
      if (S > 1) {
        a.tail_split = S;
        a.n_main = units - R;
        a.idesc_tail = idesc_f16(2 * kBlockM, p.bn / S, p.precision == 1 ? 1u : 0u);
      }
    }
  } else {
    const int tiles = a.num_m_tiles * a.num_n_tiles;
    grid = tiles < device_sm_count() ? tiles : device_sm_count();
  }
  KernelFn fn = reinterpret_cast<KernelFn>(p.fn);
  launch_pdl(fn, dim3(grid), dim3(kGemmThreads), p.smem_bytes, stream, p.maps, a);
}

}  // namespace hmi_b200

// ---------------------------------------------------------------------------
// C ABI: standalone probe
// ---------------------------------------------------------------------------
extern "C" int hmi_gpu_gemm_probe(int device, int M, int N, int K, int groups,
                                  const uint16_t* a16, const uint16_t* b16, const float* bias,
                                  const int32_t* tile_slot, const uint16_t* res0,
                                  const uint16_t* res1, int epi, int bn, int precision,
                                  void* out, float* elapsed_ms) {
  const bool cta2 = (epi & 256) != 0;  // probe flag: request the cta_group::2 kernel
  const bool no_tail = (epi & 8192) != 0;  // probe flag: no wave-tail sub-tiles
  const bool dec = (epi & 16384) != 0;     // probe flag: decode K-split cluster kernel
  epi &= ~(256 | 8192 | 16384);
  using namespace hmi_b200;
  void *dA = nullptr, *dB = nullptr, *dBias = nullptr, *dC = nullptr, *dSlot = nullptr,
       *dR0 = nullptr, *dR1 = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  int status = HMI_OK;
  try {
    HMI_CHECK(M > 0 && N > 0 && K > 0 && groups > 0, HMI_DIMENSION_ERROR, "gemm probe: sizes");
    HMI_CUDA(cudaSetDevice(device));
    const size_t out_elem = (epi & kEpiOutF32) ? 4 : 2;
    HMI_CUDA(cudaMalloc(&dA, size_t(M) * K * 2));
    HMI_CUDA(cudaMalloc(&dB, size_t(groups) * N * K * 2));
    HMI_CUDA(cudaMalloc(&dBias, size_t(groups) * N * 4));
    HMI_CUDA(cudaMalloc(&dC, size_t(M) * N * out_elem));
    HMI_CUDA(cudaMemcpy(dA, a16, size_t(M) * K * 2, cudaMemcpyHostToDevice));
    HMI_CUDA(cudaMemcpy(dB, b16, size_t(groups) * N * K * 2, cudaMemcpyHostToDevice));
    HMI_CUDA(cudaMemcpy(dBias, bias, size_t(groups) * N * 4, cudaMemcpyHostToDevice));
    HMI_CUDA(cudaMemset(dC, 0, size_t(M) * N * out_elem));
    if (tile_slot) {
      HMI_CUDA(cudaMalloc(&dSlot, size_t(M / 128) * 4));
      HMI_CUDA(cudaMemcpy(dSlot, tile_slot, size_t(M / 128) * 4, cudaMemcpyHostToDevice));
    }
    if (res0) {
      HMI_CUDA(cudaMalloc(&dR0, size_t(M) * N * 2));
      HMI_CUDA(cudaMemcpy(dR0, res0, size_t(M) * N * 2, cudaMemcpyHostToDevice));
    }
    if (res1) {
      HMI_CUDA(cudaMalloc(&dR1, size_t(M) * N * 2));
      HMI_CUDA(cudaMemcpy(dR1, res1, size_t(M) * N * 2, cudaMemcpyHostToDevice));
    }
    GemmSpec s{};
    s.a = dA; s.a_rows = M; s.a_ld = K; s.K = K;
    s.b = dB; s.N = N; s.groups = groups; s.b_ld = K;
    s.b_group_stride_bytes = size_t(N) * K * 2;
    s.bias = static_cast<const float*>(dBias); s.bias_group_stride = N;
    s.tile_slot = static_cast<const int*>(dSlot);
    s.res0 = dR0; s.res1 = dR1; s.res_ld = N;
    s.c = dC; s.c_ld = N;
    s.epi = epi; s.precision = precision; s.cta2 = cta2;
    HMI_CUDA(cudaEventCreate(&e0));
    HMI_CUDA(cudaEventCreate(&e1));
    if (dec) {  // bn = (ks << 16) | tile width, or 0: the plan's own choice
      const DecGemmCfg force{bn & 0xffff, bn >> 16};
      DecGemmPlan p = make_dec_gemm_plan(s, M / kBlockM, force);
      launch_dec_gemm(p, M, 0);
      HMI_CUDA(cudaEventRecord(e0, 0));
      launch_dec_gemm(p, M, 0);
      HMI_CUDA(cudaEventRecord(e1, 0));
    } else {
      s.bn = bn;
      GemmPlan p = make_gemm_plan(s);
      if (no_tail) p.tail_enabled = false;
      launch_gemm(p, M, 0);  // warm-up / first launch
      HMI_CUDA(cudaEventRecord(e0, 0));
      launch_gemm(p, M, 0);
      HMI_CUDA(cudaEventRecord(e1, 0));
    }
    HMI_CUDA(cudaEventSynchronize(e1));
    if (elapsed_ms) HMI_CUDA(cudaEventElapsedTime(elapsed_ms, e0, e1));
    HMI_CUDA(cudaMemcpy(out, dC, size_t(M) * N * out_elem, cudaMemcpyDeviceToHost));
  } catch (const HmiError& e) {
    set_last_error(e.what());
    status = e.code;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    status = HMI_CUDA_ERROR;
  }
  if (e0) cudaEventDestroy(e0);
  if (e1) cudaEventDestroy(e1);
  for (void* p : {dA, dB, dBias, dC, dSlot, dR0, dR1}) {
    if (p) cudaFree(p);
  }
  return status;
}

// ---------------------------------------------------------------------------
// C ABI: host -> HBM copy probe (adapter slot transfers): n pieces of `bytes` each from
// pinned host memory into scattered device slots. mode 0: one contiguous copy of n * bytes;
// 1: n cudaMemcpyAsync; 3: zero-copy gather kernel (device reads
// mapped pinned memory, `ctas` CTAs). Returns GB/s of the timed (second) repetition.
// ---------------------------------------------------------------------------
namespace {
__global__ void zero_copy_gather_kernel(const uint4* const* src, uint4* const* dst, int n,
                                        size_t vec_per_piece) {
  const size_t total = static_cast<size_t>(n) * vec_per_piece;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const size_t p = i / vec_per_piece, o = i - p * vec_per_piece;
    dst[p][o] = src[p][o];
  }
}
}  // namespace

extern "C" int hmi_gpu_copy_probe(int device, int n, size_t bytes, int mode, int ctas,
                                  double* gbps) {
  using namespace hmi_b200;
  uint8_t *h = nullptr, *dbuf = nullptr;
  void **d_src = nullptr, **d_dst = nullptr;
  cudaStream_t st = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  int status = HMI_OK;
  try {
    HMI_CHECK(mode == 0 || mode == 1 || mode == 3, HMI_CONFIG_ERROR, "copy probe: mode 0, 1 or 3");
    HMI_CUDA(cudaSetDevice(device));
    HMI_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    HMI_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&h), static_cast<size_t>(n) * bytes, cudaHostAllocMapped));
    std::memset(h, 1, static_cast<size_t>(n) * bytes);
    HMI_CUDA(cudaMalloc(&dbuf, static_cast<size_t>(2 * n) * bytes));
    std::vector<void*> src(n), dst(n), hs(n);
    for (int i = 0; i < n; ++i) {
      hs[i] = h + static_cast<size_t>(i) * bytes;
      dst[i] = dbuf + static_cast<size_t>((i * 7919) % (2 * n)) * bytes;  // scattered slots
      void* dp = nullptr;
      HMI_CUDA(cudaHostGetDevicePointer(&dp, hs[i], 0));
      src[i] = dp;
    }
    HMI_CUDA(cudaMalloc(&d_src, n * sizeof(void*)));
    HMI_CUDA(cudaMalloc(&d_dst, n * sizeof(void*)));
    HMI_CUDA(cudaMemcpy(d_src, src.data(), n * sizeof(void*), cudaMemcpyHostToDevice));
    HMI_CUDA(cudaMemcpy(d_dst, dst.data(), n * sizeof(void*), cudaMemcpyHostToDevice));
    HMI_CUDA(cudaEventCreate(&e0));
    HMI_CUDA(cudaEventCreate(&e1));
    float ms = 0.f;
    for (int rep = 0; rep < 2; ++rep) {
      HMI_CUDA(cudaEventRecord(e0, st));
      if (mode == 0) {
        HMI_CUDA(cudaMemcpyAsync(dbuf, h, static_cast<size_t>(n) * bytes, cudaMemcpyHostToDevice, st));
      } else if (mode == 1) {
        for (int i = 0; i < n; ++i)
          HMI_CUDA(cudaMemcpyAsync(dst[i], hs[i], bytes, cudaMemcpyHostToDevice, st));
      } else {
        zero_copy_gather_kernel<<<ctas, 512, 0, st>>>(reinterpret_cast<const uint4* const*>(d_src),
                                                      reinterpret_cast<uint4* const*>(d_dst), n,
                                                      bytes / 16);
        HMI_CUDA(cudaGetLastError());
      }
      HMI_CUDA(cudaEventRecord(e1, st));
      HMI_CUDA(cudaEventSynchronize(e1));
      HMI_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    }
    if (gbps) *gbps = static_cast<double>(n) * bytes / (ms * 1e-3) / 1e9;
  } catch (const HmiError& e) {
    set_last_error(e.what());
    status = e.code;
  }
  if (e0) cudaEventDestroy(e0);
  if (e1) cudaEventDestroy(e1);
  if (d_src) cudaFree(d_src);
  if (d_dst) cudaFree(d_dst);
  if (dbuf) cudaFree(dbuf);
  if (h) cudaFreeHost(h);
  if (st) cudaStreamDestroy(st);
  return status;
}
