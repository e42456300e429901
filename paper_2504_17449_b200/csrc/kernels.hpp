// SPDX-License-Identifier: Apache-2.0
// Launchers of the non-GEMM hot-path kernels (K3-K7).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "host_util.hpp"

namespace hmi_b200 {

constexpr uint32_t kNoParent = 0xffffffffu;
constexpr int kMaxNgram = 5;
constexpr uint32_t kEmptyKey = 0xffffffffu;

// One open-addressing slot of the device PLOT hash (32 B):
//   {version, key_len, t0..t4, row_base}; version == kEmptyKey marks an empty slot.
struct PlotSlot {
  uint32_t version, len, tok[kMaxNgram], row_base;
};

__host__ __device__ inline uint64_t plot_hash(uint32_t version, uint32_t len, const uint32_t* t) {
  uint64_t h = 0x9e3779b97f4a7c15ULL ^ (static_cast<uint64_t>(version) << 32 | len);
  for (uint32_t i = 0; i < len; ++i) {
    h ^= t[i] + 0x9e3779b97f4a7c15ULL + (h << 6) + (h >> 2);
    h *= 0xbf58476d1ce4e5b9ULL;
  }
  h ^= h >> 31;
  h *= 0x94d049bb133111ebULL;
  h ^= h >> 29;
  return h;
}

struct PlotDev {
  const PlotSlot* slots = nullptr;
  uint64_t mask = 0;               // capacity - 1 (power of two)
  const int32_t* parent = nullptr; // [max_versions], -1 = root / none, -2 = not a version
  int max_versions = 0;
  const float* reps = nullptr;     // [rows][d] f32, float32-exact PLOT values
  int ngram = 3;
  int d = 0;
  int max_depth = 1;               // longest version chain (branch -> ... -> root), <= 8
};

// K5: on-device PLOT retrieval (retrieve_sequence, proj/src/plot/retrieval.cpp:82-124).
void launch_retrieve(const PlotDev& plot, const uint32_t* tokens, const int* lens,
                     const int* req_version, int n_req, int S, int causal, void* h16,
                     int precision, double* h64_debug, int32_t* gather, int32_t* levels,
                     int32_t* err, cudaStream_t stream, const int32_t* dec_pos = nullptr,
                     int tok_stride = 0);

// Per-batch inputs into their device buffers with SM loads (instance ids, tokens with a source
// row stride, lengths, slot-table deltas; the error word zeroed). Sources may be pinned host
// memory (read over PCIe through unified addressing) or device memory. Unlike cudaMemcpyAsync
// this never queues behind the copy engine's adapter transfers of later batches.
struct FetchArgs {
  const uint32_t* inst = nullptr;   uint32_t* d_inst = nullptr;   int n_inst = 0;
  const uint32_t* tokens = nullptr; uint32_t* d_tokens = nullptr; int n_req = 0, S = 0, src_stride = 0;
  const int32_t* lens = nullptr;    int32_t* d_lens = nullptr;
  const int32_t* delta = nullptr;   int32_t* d_delta = nullptr;   int n_delta = 0;
  int32_t* d_err = nullptr;
};
void launch_fetch_inputs(const FetchArgs& a, cudaStream_t stream);

// Streaming PLT1 ingest: segment s = {byte offset of its rep rows in the raw chunk, dst row
// (low 31 bits), dst row (high bits), rows}; copies rows x d f32 from the chunk to dst rows.
void launch_scatter_rows(const uint8_t* chunk, const int4* segs, int n_seg, float* dst, int d,
                         cudaStream_t stream);

// K6: routing instance -> (version, task, head) and task -> per-layer HBM slot.
void launch_route(const uint32_t* instance_idx, int n_req, const int32_t* inst_version,
                  const int32_t* inst_task, const int32_t* inst_head, int n_instances,
                  const int32_t* slot_of, int layers, int tiles_per_req, int tile_stride,
                  int32_t* req_version, int32_t* req_task, int32_t* req_head,
                  int32_t* tile_slot, int32_t* err, cudaStream_t stream);

// K3 fast path for padded length 128: persistent, TMA double-buffered (request, head) items.
struct AttnPlan {
  CUtensorMap map_qkv, map_ctx;
  int d = 0;
  int precision = 0;
};
AttnPlan make_attention_plan(const void* qkv, void* ctx, int max_rows, int d, int precision);
// Same, on tcgen05 (S and O in TMEM, softmax warps write P to smem): attention_tc.cu
void launch_attention_tc(const AttnPlan& p, const int* lens, int n_req, int heads, int causal,
                         cudaStream_t stream);
// Padded lengths 256..512 on tcgen05 (two-pass softmax over 128-key blocks): attention_tc.cu
bool attention_long_tc_ok(int S);
void launch_attention_long_tc(const AttnPlan& p, const int* lens, int n_req, int S, int heads,
                              int causal, cudaStream_t stream);

// K3: attention core.
void launch_attention(const void* qkv, void* ctx, const int* lens, int n_req, int S, int d,
                      int heads, int causal, int precision, cudaStream_t stream);

// K4: LayerNorm over f32 rows (the residual sum is produced by the GEMM epilogue).
// n_parts > 0: y holds n_parts split-K partials (part_stride floats apart); the row is
// their sum + bias + res16 (16-bit) before normalising (the split GEMM's reduction)
void launch_layernorm(const float* y, const float* gamma, const float* beta, void* out16,
                      float* out32, int rows, int d, int precision, cudaStream_t stream,
                      int n_parts = 0, long long part_stride = 0, const float* bias = nullptr,
                      const void* res16 = nullptr);

// K7: per-request task head + first-max argmax (apply_head, model.cpp:120-171).
struct HeadDev {
  const float* arena = nullptr;     // all heads, f32
  const int64_t* offset = nullptr;  // [heads] float offset of W (d x labels) ; b follows
  const int32_t* labels = nullptr;  // [heads]
  const int32_t* kind = nullptr;    // [heads] 0 cls, 1 token_tag, 2 lm
  // LN folding: rows come pre-norm (16-bit) and the head applies LayerNorm exactly (f64)
  const void* y16 = nullptr;
  const float* ln_g = nullptr;
  const float* ln_b = nullptr;
  int bf16 = 0;
};

// Final LayerNorm of pre-norm 16-bit rows from partial statistics (debug / introspection).
void launch_normalize_rows(const void* y16, const float2* stats, int n_part, float inv_n,
                           const float* gamma, const float* beta, float* out, int rows, int d,
                           int precision, cudaStream_t stream);
void launch_head(const HeadDev& heads, const float* h32, const int32_t* req_head,
                 const int* lens, int n_req, int S, int d, int max_labels, float* scores,
                 int32_t* labels_out, int32_t* tags, cudaStream_t stream);

}  // namespace hmi_b200
