// SPDX-License-Identifier: Apache-2.0
// Host interface of the tcgen05 GEMM (K1/K2). See gemm_tcgen05.cuh for the kernel.
#pragma once

#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "host_util.hpp"

namespace hmi_b200 {

// Kernel-side arguments (passed by value).
struct GemmArgs {
  int M, N, K;                 // N is per-group
  int num_m_tiles, num_n_tiles;
  const float* bias;           // [N] (+ group * bias_slot_stride floats)
  long long bias_slot_stride;  // in floats, 0 when weights are shared
  const int* tile_slot;        // per M tile group index (nullptr: group 0)
  const __half* res0;          // optional residual inputs, row-major ld = res_ld (16-bit)
  const __half* res1;
  int res_ld;
  uint32_t idesc;
  // --- LayerNorm folding (kEpiStats / kEpiFoldLN / kEpiRes0LN / kEpiRes1LN) ---
  float2* stats_out;           // kEpiStats: per (row, n tile, column half) (sum, sum of squares)
  int stats_ld;                // float2 entries per row
  const float2* a_stats;       // kEpiFoldLN: partial stats of A's (pre-norm) rows
  int a_stats_n;               // partials per row
  const float* colsum;         // kEpiFoldLN: sum_k of the gamma-folded 16-bit weights, per column
  const float2* r_stats;       // kEpiRes0LN/kEpiRes1LN: partial stats of the pre-norm residual
  int r_stats_n;
  const float* r_gamma;        // LayerNorm applied on the fly to that residual
  const float* r_beta;
  float inv_n;                 // 1 / (row width the statistics cover)
  // pair kernel wave-tail split: units [0, n_main) run whole; each of the remaining units is
  // cut into tail_split narrower N sub-tiles (MMA N = BN / tail_split, idesc_tail) so the last
  // partial wave spreads over more SMs. Per-element K order is unchanged (bit-identical).
  int n_main;
  int tail_split;
  uint32_t idesc_tail;
  int tail_r1;                 // tail B boxes through maps.r1 (else maps.r0)
  // tenant extension (kEpiExt, pair kernel): after the K / 64 shared blocks, 2 x ext_kb more
  // per unit. Block (e, k) multiplies the ext rows (maps.xa: the bottleneck activations mid,
  // [rows][64 ext_kb]) of pair tile e -- zero rows (ext_zero_row) in the other CTA's half -- by
  // tile e's tenant slot (maps.xb: Wu^T [N][64 ext_kb] per slot), so the two requests of a
  // 256-row pair unit each meet their own up projection. The epilogue adds bias2 of the CTA
  // tile's slot (b_u).
  int ext_kb;
  int ext_zero_row;
  const float* bias2;
  long long bias2_stride;      // floats per slot
  // device-side readiness wait before the first operand load (1-CTA grouped kernel, fine
  // pipeline): proceed once *ready - ready_seq (wrap-safe) is non-negative; err latches
  // HMI_SCHEDULING_BUG if the flag never comes
  const uint32_t* ready;
  uint32_t ready_seq;
  int32_t* err;
};

// Epilogue flags
constexpr int kEpiRelu = 1;
constexpr int kEpiRes1 = 2;  // add res0
constexpr int kEpiRes2 = 4;  // add res0 + res1
constexpr int kEpiOutF32 = 8;
constexpr int kEpiBf16 = 16;  // 16-bit outputs / residuals are bf16 (set from precision)
constexpr int kEpiResTma = 128;  // 1-CTA, two residuals: residual tiles TMA-staged in smem
// LayerNorm folding: LN(y) is never materialised; its consumers apply it.
constexpr int kEpiStats = 256;   // write per-row partial (sum, sumsq) of the output, one per
                                 // 64-column group (16-bit outputs only)
constexpr int kStatsStride = 16; // float2 entries per row of a partial-statistics buffer
constexpr int kEpiFoldLN = 512;  // A is pre-norm y: out = inv*(acc - mean*colsum) + bias
constexpr int kEpiRes0LN = 1024; // residual res0 is pre-norm: add LN(res0) (r_* args)
constexpr int kEpiRes1LN = 2048; // residual res1 is pre-norm: add LN(res1)
constexpr int kEpiExt = 4096;    // pair kernel: tenant extension blocks + bias2 (see GemmArgs)

// All tensor maps of one GEMM (passed as one __grid_constant__ kernel parameter).
struct GemmMaps {
  CUtensorMap a, b, c, r0, r1;
  CUtensorMap xa, xb, xb0, xb1;  // kEpiExt: ext rows, tenant B (main / tail widths r0 / r1)
  CUtensorMap res;               // pair kernel, one 16-bit residual: 64 x 32 boxes of res0
};

// Everything needed to bind one GEMM to fixed device buffers.
struct GemmSpec {
  const void* a = nullptr;  // [a_rows][a_ld] 16-bit
  int a_rows = 0, a_ld = 0, K = 0;
  const void* b = nullptr;  // [groups][N][b_ld] 16-bit
  int N = 0, groups = 1, b_ld = 0;
  size_t b_group_stride_bytes = 0;
  const float* bias = nullptr;       // [groups][bias_group_stride]
  long long bias_group_stride = 0;   // floats
  const int* tile_slot = nullptr;    // per 128-row tile group index (device), or null
  const void* res0 = nullptr;        // 16-bit residuals [rows][res_ld]
  const void* res1 = nullptr;
  int res_ld = 0;
  void* c = nullptr;                 // output [a_rows][c_ld], 16-bit or f32
  int c_ld = 0;
  int epi = 0;                       // kEpi* flags
  int bn = 256;                      // N tile
  int precision = 0;                 // 0 fp16, 1 bf16
  bool cta2 = false;                 // cta_group::2 pair kernel (shared weights only)
  float2* stats_out = nullptr;       // kEpiStats
  int stats_ld = 0;
  const float2* a_stats = nullptr;   // kEpiFoldLN
  int a_stats_n = 0;
  const float* colsum = nullptr;
  const float2* r_stats = nullptr;   // kEpiRes0LN / kEpiRes1LN
  int r_stats_n = 0;
  const float* r_gamma = nullptr;
  const float* r_beta = nullptr;
  float inv_n = 0.f;
  // kEpiExt (pair kernel): ext rows [a_rows + 128][ext_k] 16-bit whose last 128 rows are zero,
  // tenant B [slots][N][ext_b_ld] at ext_b (slot stride ext_b_stride bytes), tenant bias
  // ext_bias + slot * ext_bias_stride; the slot of each 128-row tile is tile_slot[tile]
  const void* ext_a = nullptr;
  int ext_k = 0;
  const void* ext_b = nullptr;
  int ext_b_ld = 0, ext_groups = 0;
  size_t ext_b_stride = 0;
  const float* ext_bias = nullptr;
  long long ext_bias_stride = 0;
};

struct GemmPlan {
  GemmMaps maps;
  GemmArgs args;
  void* fn = nullptr;
  int smem_bytes = 0;
  int max_rows = 0;
  bool two_cta = false;
  int tail_s0 = 0, tail_s1 = 0;  // pair kernel: tail splits served by maps.r0 / maps.r1 (0: none)
  bool tail_enabled = true;      // the GEMM test entry point can disable the wave-tail split
  int precision = 0, bn = 0;
  int max_clusters = 0;  // pair kernel: co-resident CTA pairs (cudaOccupancyMaxActiveClusters)
};

GemmPlan make_gemm_plan(const GemmSpec& s);

// Decode-step GEMM (gemm_dec.cu): one 128 x bn tile per cluster of ks CTAs, each CTA one
// K / ks slice, partials reduced through distributed shared memory. Epilogues: bias,
// bias + ReLU, bias -> f32, bias + res0 -> f32.
struct DecGemmArgs {
  int num_n_tiles, ks, kb_per_cta;
  const float* bias;
  const void* res0;  // 16-bit [rows][res_ld]
  int res_ld;
  void* c;           // 16-bit or f32 [rows][c_ld]
  int c_ld;
  uint32_t idesc;
};
struct DecGemmMaps {
  CUtensorMap a, b;
};
struct DecGemmCfg {
  int bn, ks;
};
struct DecGemmPlan {
  DecGemmMaps maps;
  DecGemmArgs args;
  DecGemmCfg cfg{0, 0};
  void* fn = nullptr;
  int smem_bytes = 0;
  int max_rows = 0;
};
DecGemmCfg pick_dec_cfg(int N, int K, int m_tiles, int sms, int epi);
DecGemmPlan make_dec_gemm_plan(const GemmSpec& s, int m_tiles, DecGemmCfg force = {0, 0});
void launch_dec_gemm(const DecGemmPlan& p, int M, cudaStream_t stream);
void launch_gemm(const GemmPlan& p, int M, cudaStream_t stream, const uint32_t* ready = nullptr,
                 uint32_t ready_seq = 0, int32_t* err = nullptr);

}  // namespace hmi_b200
