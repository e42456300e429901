// SPDX-License-Identifier: Apache-2.0
// GPU PLOT builder: lower_stack_forward on the tcgen05 GEMM + build_root / derive_branch
// key selection on the host (proj/src/plot/table.cpp:16-104).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <vector>

#include "host_util.hpp"

namespace hmi_b200 {

// ingest.cpp: one-pass ADP1 read with the model's dimensions expected
void load_adp1_expect(const char* path, uint32_t L, uint32_t D, uint32_t R, float* body);

constexpr int kMaxFragment = 5;

void launch_plot_embed(const float* tok_emb, const float* pos_emb, const uint32_t* keys, int ngram,
                       int k, int n, int rows, int d, void* h16, int precision, cudaStream_t stream);
void launch_plot_attention(const void* qkv, void* ctx, int k, int n, int heads, int d, int causal,
                           int precision, cudaStream_t stream);

using NGramKey = std::vector<uint32_t>;
// std::map order over keys = the reference's PlotTable::entries order (table.hpp, PLT1 order)
using CountMap = std::map<NGramKey, uint64_t>;

// count_kgrams (table.cpp:16-27)
CountMap count_kgrams(uint32_t n_seq, const uint32_t* seq_lens, const uint32_t* tokens, uint32_t k);
// build_root's key set (table.cpp:29-58): every k-gram, k = 1..ngram, plus the vocabulary-wide
// uni-gram backstop with frequency 1
CountMap select_root(uint32_t n_seq, const uint32_t* seq_lens, const uint32_t* tokens,
                     uint32_t ngram, uint32_t vocab);
// derive_branch's key set (table.cpp:60-104): ngram-grams by count descending (ties in key
// order) until cumulative / total >= alpha
CountMap select_branch(uint32_t n_seq, const uint32_t* seq_lens, const uint32_t* tokens,
                       uint32_t ngram, double alpha_percent);

}  // namespace hmi_b200

// Opaque C-ABI handles (include/hmi_gpu.h)
struct hmi_plot_table {
  uint32_t ngram = 0, d = 0;
  std::vector<uint32_t> key_len;  // [n]
  std::vector<uint32_t> keys;     // [n][ngram], zero padded
  std::vector<uint64_t> freq;     // [n]
  std::vector<float> reps;        // [sum key_len][d] (empty for a key selection only)
};
