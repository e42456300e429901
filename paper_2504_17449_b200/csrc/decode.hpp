// SPDX-License-Identifier: Apache-2.0
// Launchers of the causal-generation kernels (decode.cu).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "host_util.hpp"

namespace hmi_b200 {

// Final row of each request -> f32 (rescoring) + 16-bit (lm GEMM operand). y16 non-null:
// the rows are pre-norm and LayerNorm(gamma, beta) is applied in f64; else h32 is copied.
void launch_lm_gather(const void* y16, const float* h32, const float* gamma, const float* beta,
                      const int* lens, int n_req, int S, int d, int precision, float* out32,
                      void* out16, cudaStream_t stream);

struct LmArgmaxArgs {
  const float* logits = nullptr;  // [n][ld] f32 from the lm GEMM
  int ld = 0;
  int V = 0;                      // real vocabulary (columns >= V are padding)
  const float* h32 = nullptr;     // [n][d] f32 final rows
  int d = 0;
  const float* w = nullptr;       // [d][V] f32 head weights (reference layout)
  const float* wT = nullptr;      // optional [V][d] f32 transpose (coalesced candidate reads)
  const float* bias = nullptr;    // [V] f32
  const int32_t* req_head = nullptr;  // optional: only requests bound to `head`
  int head = -1;
  int32_t* labels_out = nullptr;  // [n]
  float* scores_out = nullptr;    // [n][scores_ld], column 0 = the chosen logit
  int scores_ld = 0;
  // generation (optional): append the token to the sequence
  uint32_t* gen_tokens = nullptr;  // [n][tok_stride]
  int tok_stride = 0;
  int32_t* gen_pos = nullptr;      // [n]
  int advance = 0;                 // 1: gen_pos += 1 before writing
  int32_t* out_tokens = nullptr;   // [n][out_ld]
  float* out_logits = nullptr;     // [n][out_ld]
  int out_ld = 0;
  int step = 0;                    // output column; < 0: gen_pos (after advance) - lens[b], so
  const int* lens = nullptr;       // one launch serves every step (CUDA-graph replay)
};
void launch_lm_argmax(const LmArgmaxArgs& a, int n_req, cudaStream_t stream);

struct AttnDecodeArgs {
  const uint16_t* qkv_new = nullptr;      // [n][3d] this step's projections
  const uint16_t* qkv_prefill = nullptr;  // [n * S][3d] the prompt's projections (this layer)
  int S = 0;                              // prompt padded length
  uint16_t* tail = nullptr;               // [n][tail_cap][2d] generated rows' k | v (this layer)
  int tail_cap = 0;
  const int* lens = nullptr;              // prompt lengths
  const int32_t* gen_pos = nullptr;       // position of the new row
  uint16_t* ctx = nullptr;                // [n][d]
  int d = 0;
  float scale = 0.f;
  int bf16 = 0;
};
void launch_attn_decode(const AttnDecodeArgs& a, int n_req, int heads, int max_keys,
                        cudaStream_t stream);

// TMA-staged form (one layer): the request's prompt K / V head slices (SWIZZLE_128B boxes of
// 128 rows x 64 dims over the layer's prompt q|k|v buffer) and its generated rows' k / v (one
// box of tail_cap rows over the layer's tail buffer) land in shared memory with four bulk
// copies; scores and context then read shared memory only.
struct AttnDecodeMaps {
  CUtensorMap prefill;  // [rows][3d] 16-bit, box 64 x 128
  CUtensorMap tail;     // [n * tail_cap][2d] 16-bit, box 64 x tail_cap
};
bool attn_decode_tma_ok(int S, int tail_cap);
AttnDecodeMaps make_attn_decode_maps(const void* qkv_prefill, int max_rows, void* tail,
                                     int max_batch, int tail_cap, int d, int precision);
void launch_attn_decode_tma(const AttnDecodeArgs& a, const AttnDecodeMaps& m, int n_req,
                            int heads, cudaStream_t stream);

struct AdapterRowsArgs {
  const uint16_t* ctx16 = nullptr;  // [n][d] attention context (input of the folded down proj.)
  const uint16_t* a16 = nullptr;  // [n][d] attention output (after Wo, bo)
  const uint16_t* h16 = nullptr;  // [n][d] layer input (residual)
  const int32_t* req_task = nullptr;
  const int32_t* slot_of = nullptr;  // [task][layers]
  int layers = 0, layer = 0;
  const uint8_t* arena = nullptr;
  size_t slot_bytes = 0;
  int d = 0, r_pad = 0;
  const float* ln_g = nullptr;
  const float* ln_b = nullptr;
  uint16_t* x16 = nullptr;  // [n][d] LN1 output
  int32_t* err = nullptr;
  int bf16 = 0;
};
void launch_adapter_rows_ln(const AdapterRowsArgs& a, int n_req, cudaStream_t stream);

}  // namespace hmi_b200
