// SPDX-License-Identifier: Apache-2.0
//
// GPU PLOT builder: the offline table construction of the reference,
//
//   build_root     (proj/src/plot/table.cpp:29-58)   every k-gram of the corpus (k = 1..n) plus
//                                                    the vocabulary-wide uni-gram backstop
//   derive_branch  (proj/src/plot/table.cpp:60-104)  the domain corpus' n-grams by count until
//                                                    the alpha share of occurrences is covered
//
// with each selected key's representation = lower_stack_forward (model.cpp:96-118) computed on
// the GPU: fragments of equal length are packed into 128-row tiles (fragment f, position i at
// row f * len + i) and run through the lower layers with the same tcgen05 GEMM as the serving
// path (QKV, O + residual, FFN1 + ReLU, FFN2 + residual), the K4 LayerNorm kernel and a
// fragment attention kernel (plot_kernels.cu). Key selection is exact host integer logic over
// std::map (the reference's entry order), so keys and frequencies match it bit for bit.
#include "plot_builder.hpp"

#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>

#include "gemm.hpp"
#include "kernels.hpp"

namespace hmi_b200 {

CountMap count_kgrams(uint32_t n_seq, const uint32_t* seq_lens, const uint32_t* tokens, uint32_t k) {
  CountMap counts;
  const uint32_t* t = tokens;
  for (uint32_t s = 0; s < n_seq; ++s) {
    const uint32_t len = seq_lens[s];
    if (len >= k) {
      for (uint32_t i = 0; i + k <= len; ++i) counts[NGramKey(t + i, t + i + k)] += 1;
    }
    t += len;
  }
  return counts;
}

CountMap select_root(uint32_t n_seq, const uint32_t* seq_lens, const uint32_t* tokens,
                     uint32_t ngram, uint32_t vocab) {
  HMI_CHECK(n_seq > 0, HMI_BUILD_ERROR, "cannot build a table from an empty corpus");
  CountMap entries;
  for (uint32_t k = 1; k <= ngram; ++k) {
    for (auto& [key, freq] : count_kgrams(n_seq, seq_lens, tokens, k)) entries.emplace(key, freq);
  }
  for (uint32_t t = 0; t < vocab; ++t) entries.emplace(NGramKey{t}, 1);  // kept if present
  return entries;
}

CountMap select_branch(uint32_t n_seq, const uint32_t* seq_lens, const uint32_t* tokens,
                       uint32_t ngram, double alpha_percent) {
  HMI_CHECK(alpha_percent >= 0.0 && alpha_percent <= 100.0, HMI_CONFIG_ERROR,
            "alpha_percent must be in [0, 100]");
  const uint64_t alpha_centi = static_cast<uint64_t>(std::llround(alpha_percent * 100.0));
  const CountMap counts = count_kgrams(n_seq, seq_lens, tokens, ngram);
  uint64_t total = 0;
  for (const auto& kv : counts) total += kv.second;
  CountMap out;
  if (total == 0 || alpha_centi == 0) return out;
  std::vector<const CountMap::value_type*> order;
  order.reserve(counts.size());
  for (const auto& kv : counts) order.push_back(&kv);
  std::stable_sort(order.begin(), order.end(),
                   [](const auto* a, const auto* b) { return a->second > b->second; });
  uint64_t cumulative = 0;
  for (const auto* kv : order) {
    cumulative += kv->second;
    out.emplace(kv->first, kv->second);
    if (cumulative * 10000 >= alpha_centi * total) break;  // exact integer alpha test
  }
  return out;
}

namespace {

uint16_t to16(float x, int precision) {
  if (precision == 1) {
    __nv_bfloat16 b = __float2bfloat16_rn(x);
    return *reinterpret_cast<uint16_t*>(&b);
  }
  __half h = __float2half_rn(x);
  return *reinterpret_cast<uint16_t*>(&h);
}

template <typename T>
T* dev_alloc(size_t n) {
  T* p = nullptr;
  if (n) HMI_CUDA(cudaMalloc(&p, n * sizeof(T)));
  return p;
}

struct LowerLayer {
  uint16_t *wqkv = nullptr, *wo = nullptr, *w1 = nullptr, *w2 = nullptr;  // [out][in] 16-bit
  float *bqkv = nullptr, *bo = nullptr, *b1 = nullptr, *b2 = nullptr;
  float *ln1g = nullptr, *ln1b = nullptr, *ln2g = nullptr, *ln2b = nullptr;
  GemmPlan qkv, oproj, ffn1, ffn2;
};

}  // namespace

struct PlotBuilder {
  int device = 0, precision = 0;
  hmi_model_config cfg{};
  int d = 0, f = 0, max_rows = 0;
  std::vector<void*> allocs;
  float *tok_emb = nullptr, *pos_emb = nullptr;
  std::vector<LowerLayer> layers;
  uint32_t* keys_d = nullptr;
  uint16_t *h16 = nullptr, *qkv16 = nullptr, *ctx16 = nullptr, *x16 = nullptr, *ffn16 = nullptr;
  float *y32 = nullptr, *out32 = nullptr;
  // pinned staging, double-buffered: fragment keys in, f32 rows out
  uint32_t* keys_pin[2] = {nullptr, nullptr};
  float* out_pin[2] = {nullptr, nullptr};
  cudaEvent_t ev0[2] = {}, ev1[2] = {}, done[2] = {};
  double device_ms = 0.0;
  uint64_t rows_done = 0;
  cudaStream_t stream = nullptr;
  std::mutex mu;

  template <typename T>
  T* alloc(size_t n) {
    T* p = dev_alloc<T>(n);
    allocs.push_back(p);
    return p;
  }

  ~PlotBuilder() {
    for (void* p : allocs) cudaFree(p);
    for (int i = 0; i < 2; ++i) {
      if (keys_pin[i]) cudaFreeHost(keys_pin[i]);
      if (out_pin[i]) cudaFreeHost(out_pin[i]);
      for (cudaEvent_t e : {ev0[i], ev1[i], done[i]})
        if (e) cudaEventDestroy(e);
    }
    if (stream) cudaStreamDestroy(stream);
  }

  void upload_layer(const float* w, LowerLayer& L) {
    const size_t D = d, F = f;
    const float *wq = w, *bq = wq + D * D, *wk = bq + D, *bk = wk + D * D, *wv = bk + D,
                *bv = wv + D * D, *wo = bv + D, *bo = wo + D * D, *w1 = bo + D, *b1 = w1 + D * F,
                *w2 = b1 + F, *b2 = w2 + F * D, *g1 = b2 + D, *s1 = g1 + D, *g2 = s1 + D,
                *s2 = g2 + D;
    std::vector<uint16_t> t16(3 * D * D + D * D + F * D + D * F);
    auto transpose = [&](const float* src, size_t in, size_t out, uint16_t* dst) {
      for (size_t o = 0; o < out; ++o)
        for (size_t i = 0; i < in; ++i) dst[o * in + i] = to16(src[i * out + o], precision);
    };
    transpose(wq, D, D, t16.data());
    transpose(wk, D, D, t16.data() + D * D);
    transpose(wv, D, D, t16.data() + 2 * D * D);
    transpose(wo, D, D, t16.data() + 3 * D * D);
    transpose(w1, D, F, t16.data() + 4 * D * D);
    transpose(w2, F, D, t16.data() + 4 * D * D + F * D);
    uint16_t* p16 = alloc<uint16_t>(t16.size());
    HMI_CUDA(cudaMemcpy(p16, t16.data(), t16.size() * 2, cudaMemcpyHostToDevice));
    L.wqkv = p16;
    L.wo = p16 + 3 * D * D;
    L.w1 = L.wo + D * D;
    L.w2 = L.w1 + F * D;
    std::vector<float> v;
    for (const auto& [p, n] : std::vector<std::pair<const float*, size_t>>{
             {bq, D}, {bk, D}, {bv, D}, {bo, D}, {b1, F}, {b2, D}, {g1, D}, {s1, D}, {g2, D}, {s2, D}})
      v.insert(v.end(), p, p + n);
    float* p32 = alloc<float>(v.size());
    HMI_CUDA(cudaMemcpy(p32, v.data(), v.size() * 4, cudaMemcpyHostToDevice));
    L.bqkv = p32;
    L.bo = p32 + 3 * D;
    L.b1 = L.bo + D;
    L.b2 = L.b1 + F;
    L.ln1g = L.b2 + D;
    L.ln1b = L.ln1g + D;
    L.ln2g = L.ln1b + D;
    L.ln2b = L.ln2g + D;
  }

  void build_plans() {
    const int sms = device_sm_count();
    (void)sms;
    for (LowerLayer& L : layers) {
      GemmSpec s;
      s.precision = precision;
      s.a_rows = max_rows;
      s.bn = 256 <= 3 * d && (3 * d) % 256 == 0 ? 256 : 128;
      s.cta2 = true;
      // QKV
      s.a = h16; s.a_ld = d; s.K = d;
      s.b = L.wqkv; s.N = 3 * d; s.b_ld = d; s.b_group_stride_bytes = size_t(3) * d * d * 2;
      s.bias = L.bqkv; s.c = qkv16; s.c_ld = 3 * d; s.epi = 0;
      L.qkv = make_gemm_plan(s);
      // O projection + residual h -> y (f32), LN1 -> x
      s.bn = d % 256 == 0 ? 256 : 128;
      s.a = ctx16; s.b = L.wo; s.N = d; s.b_group_stride_bytes = size_t(d) * d * 2;
      s.bias = L.bo; s.res0 = h16; s.res_ld = d; s.c = y32; s.c_ld = d;
      s.epi = kEpiRes1 | kEpiOutF32;
      L.oproj = make_gemm_plan(s);
      // FFN1 (ReLU)
      s.bn = f % 256 == 0 ? 256 : 128;
      s.a = x16; s.b = L.w1; s.N = f; s.b_group_stride_bytes = size_t(f) * d * 2;
      s.bias = L.b1; s.res0 = nullptr; s.c = ffn16; s.c_ld = f; s.epi = kEpiRelu;
      L.ffn1 = make_gemm_plan(s);
      // FFN2 + residual x -> y (f32), LN2 -> h
      s.bn = d % 256 == 0 ? 256 : 128;
      s.a = ffn16; s.a_ld = f; s.K = f; s.b = L.w2; s.N = d; s.b_ld = f;
      s.b_group_stride_bytes = size_t(d) * f * 2; s.bias = L.b2; s.res0 = x16; s.res_ld = d;
      s.c = y32; s.c_ld = d; s.epi = kEpiRes1 | kEpiOutF32;
      L.ffn2 = make_gemm_plan(s);
    }
  }

  // One GPU pass: lower_stack_forward of `cnt` fragments of length k (keys [cnt][ngram] in the
  // pinned staging buffer `buf`); the f32 rows (f * k + i) are copied back into pinned out[buf]
  // and done[buf] recorded. Device time between ev0/ev1 accumulates into device_ms.
  void enqueue_pass(int buf, uint32_t k, uint32_t cnt) {
    const int ngram = static_cast<int>(cfg.max_fragment);
    const int rows = static_cast<int>(cnt * k);
    const int rows_p = (rows + 127) / 128 * 128;
    HMI_CUDA(cudaEventRecord(ev0[buf], stream));
    HMI_CUDA(cudaMemcpyAsync(keys_d, keys_pin[buf], static_cast<size_t>(cnt) * ngram * 4,
                             cudaMemcpyHostToDevice, stream));
    launch_plot_embed(tok_emb, pos_emb, keys_d, ngram, static_cast<int>(k), static_cast<int>(cnt),
                      rows_p, d, h16, precision, stream);
    const int causal = cfg.mode == 1 ? 1 : 0;
    for (size_t l = 0; l < layers.size(); ++l) {
      const LowerLayer& L = layers[l];
      const bool last = l + 1 == layers.size();
      launch_gemm(L.qkv, rows_p, stream);
      launch_plot_attention(qkv16, ctx16, static_cast<int>(k), static_cast<int>(cnt),
                            static_cast<int>(cfg.heads), d, causal, precision, stream);
      launch_gemm(L.oproj, rows_p, stream);
      launch_layernorm(y32, L.ln1g, L.ln1b, x16, nullptr, rows_p, d, precision, stream);
      launch_gemm(L.ffn1, rows_p, stream);
      launch_gemm(L.ffn2, rows_p, stream);
      launch_layernorm(y32, L.ln2g, L.ln2b, h16, last ? out32 : nullptr, rows_p, d, precision,
                       stream);
    }
    HMI_CUDA(cudaEventRecord(ev1[buf], stream));
    HMI_CUDA(cudaMemcpyAsync(out_pin[buf], out32, static_cast<size_t>(rows) * d * 4,
                             cudaMemcpyDeviceToHost, stream));
    HMI_CUDA(cudaEventRecord(done[buf], stream));
    rows_done += static_cast<uint64_t>(rows);
  }

  // reps of n fragments (key_len[i] tokens at keys[i * ngram]) in input order. Passes alternate
  // between two pinned staging buffers: the host scatters pass p's rows into `reps` while the
  // GPU runs pass p + 1.
  void forward(uint32_t n, const uint32_t* key_len, const uint32_t* keys, float* reps) {
    const uint32_t ngram = cfg.max_fragment;
    std::vector<uint64_t> off(n + 1, 0);
    for (uint32_t i = 0; i < n; ++i) {
      HMI_CHECK(key_len[i] >= 1 && key_len[i] <= ngram, HMI_DIMENSION_ERROR,
                "fragment length must be in [1, " + std::to_string(ngram) + "]");
      for (uint32_t j = 0; j < key_len[i]; ++j) {
        HMI_CHECK(keys[static_cast<size_t>(i) * ngram + j] < cfg.vocab_size, HMI_VOCABULARY_ERROR,
                  "token id " + std::to_string(keys[static_cast<size_t>(i) * ngram + j]) +
                      " outside vocabulary of " + std::to_string(cfg.vocab_size));
      }
      off[i + 1] = off[i] + key_len[i];
    }
    struct Pass {
      uint32_t k, cnt;
      std::vector<uint32_t> frags;
    };
    std::vector<Pass> passes;
    for (uint32_t k = 1; k <= ngram; ++k) {
      std::vector<uint32_t> idx;
      for (uint32_t i = 0; i < n; ++i)
        if (key_len[i] == k) idx.push_back(i);
      const uint32_t per = static_cast<uint32_t>(max_rows) / k;
      for (size_t c0 = 0; c0 < idx.size(); c0 += per) {
        const uint32_t cnt = static_cast<uint32_t>(std::min<size_t>(per, idx.size() - c0));
        passes.push_back({k, cnt, std::vector<uint32_t>(idx.begin() + c0, idx.begin() + c0 + cnt)});
      }
    }
    auto drain = [&](size_t p) {
      const int buf = static_cast<int>(p & 1);
      HMI_CUDA(cudaEventSynchronize(done[buf]));
      float ms = 0.f;
      HMI_CUDA(cudaEventElapsedTime(&ms, ev0[buf], ev1[buf]));
      device_ms += ms;
      const Pass& ps = passes[p];
      for (uint32_t j = 0; j < ps.cnt; ++j) {
        std::memcpy(reps + off[ps.frags[j]] * d, out_pin[buf] + static_cast<size_t>(j) * ps.k * d,
                    static_cast<size_t>(ps.k) * d * 4);
      }
    };
    for (size_t p = 0; p < passes.size(); ++p) {
      const int buf = static_cast<int>(p & 1);
      if (p >= 2) drain(p - 2);  // frees staging buffer `buf`
      const Pass& ps = passes[p];
      for (uint32_t j = 0; j < ps.cnt; ++j)
        std::memcpy(keys_pin[buf] + static_cast<size_t>(j) * ngram,
                    keys + static_cast<size_t>(ps.frags[j]) * ngram, ngram * 4);
      enqueue_pass(buf, ps.k, ps.cnt);
    }
    for (size_t p = passes.size() >= 2 ? passes.size() - 2 : 0; p < passes.size(); ++p) drain(p);
  }

  hmi_plot_table* materialize(const CountMap& sel) {
    auto* t = new hmi_plot_table;
    t->ngram = cfg.max_fragment;
    t->d = static_cast<uint32_t>(d);
    const size_t n = sel.size();
    t->key_len.resize(n);
    t->keys.assign(n * t->ngram, 0);
    t->freq.resize(n);
    uint64_t rows = 0;
    size_t e = 0;
    for (const auto& [key, fr] : sel) {
      t->key_len[e] = static_cast<uint32_t>(key.size());
      std::copy(key.begin(), key.end(), t->keys.begin() + e * t->ngram);
      t->freq[e] = fr;
      rows += key.size();
      ++e;
    }
    t->reps.resize(rows * d);
    try {
      forward(static_cast<uint32_t>(n), t->key_len.data(), t->keys.data(), t->reps.data());
    } catch (...) {
      delete t;
      throw;
    }
    return t;
  }
};

}  // namespace hmi_b200

struct hmi_plot_builder {
  hmi_b200::PlotBuilder impl;
};

namespace {

template <typename F>
int plot_guarded(F&& fn) {
  try {
    fn();
    return HMI_OK;
  } catch (const hmi_b200::HmiError& e) {
    hmi_b200::set_last_error(e.what());
    return e.code;
  } catch (const std::bad_alloc& e) {
    hmi_b200::set_last_error(std::string("host allocation failed: ") + e.what());
    return HMI_CAPACITY_ERROR;
  } catch (const std::exception& e) {
    hmi_b200::set_last_error(e.what());
    return HMI_CUDA_ERROR;
  }
}

}  // namespace

extern "C" {

int hmi_plot_builder_create(int device, const hmi_model_config* cfg, const float* token_emb,
                            const float* pos_emb, const float* lower_f32, uint32_t precision,
                            uint32_t max_rows, hmi_plot_builder** out) {
  using namespace hmi_b200;
  return plot_guarded([&] {
    HMI_CHECK(cfg && token_emb && pos_emb && out, HMI_CONFIG_ERROR, "null argument");
    HMI_CHECK(cfg->lower_layers >= 1 && lower_f32, HMI_BUILD_ERROR, "model has no lower stack");
    HMI_CHECK(cfg->heads > 0 && cfg->hidden_size == cfg->heads * 64, HMI_CONFIG_ERROR,
              "device path requires hidden_size / heads == 64");
    HMI_CHECK(cfg->hidden_size % 128 == 0 && cfg->ffn_size % 128 == 0, HMI_CONFIG_ERROR,
              "device path requires hidden_size and ffn_size multiples of 128");
    HMI_CHECK(cfg->max_fragment >= 1 && cfg->max_fragment <= kMaxFragment, HMI_CONFIG_ERROR,
              "max_fragment must be in [1, 5]");
    HMI_CHECK(precision <= 1, HMI_CONFIG_ERROR, "precision must be 0 (fp16) or 1 (bf16)");
    auto holder = std::make_unique<hmi_plot_builder>();
    PlotBuilder& b = holder->impl;
    b.device = device;
    b.precision = static_cast<int>(precision);
    b.cfg = *cfg;
    b.d = static_cast<int>(cfg->hidden_size);
    b.f = static_cast<int>(cfg->ffn_size);
    b.max_rows = static_cast<int>(std::max<uint32_t>(128, (max_rows ? max_rows : 16384) / 128 * 128));
    HMI_CUDA(cudaSetDevice(device));
    HMI_CUDA(cudaStreamCreateWithFlags(&b.stream, cudaStreamNonBlocking));
    const size_t d = b.d, f = b.f, R = b.max_rows;
    b.tok_emb = b.alloc<float>(static_cast<size_t>(cfg->vocab_size) * d);
    HMI_CUDA(cudaMemcpy(b.tok_emb, token_emb, static_cast<size_t>(cfg->vocab_size) * d * 4,
                        cudaMemcpyHostToDevice));
    b.pos_emb = b.alloc<float>(static_cast<size_t>(cfg->max_fragment) * d);
    HMI_CUDA(cudaMemcpy(b.pos_emb, pos_emb, static_cast<size_t>(cfg->max_fragment) * d * 4,
                        cudaMemcpyHostToDevice));
    b.keys_d = b.alloc<uint32_t>(R * cfg->max_fragment);
    b.h16 = b.alloc<uint16_t>(R * d);
    b.qkv16 = b.alloc<uint16_t>(R * 3 * d);
    b.ctx16 = b.alloc<uint16_t>(R * d);
    b.x16 = b.alloc<uint16_t>(R * d);
    b.ffn16 = b.alloc<uint16_t>(R * f);
    b.y32 = b.alloc<float>(R * d);
    b.out32 = b.alloc<float>(R * d);
    HMI_CUDA(cudaMemset(b.ctx16, 0, R * d * 2));
    for (int i = 0; i < 2; ++i) {
      HMI_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&b.keys_pin[i]), R * cfg->max_fragment * 4, 0));
      HMI_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&b.out_pin[i]), R * d * 4, 0));
      HMI_CUDA(cudaEventCreate(&b.ev0[i]));
      HMI_CUDA(cudaEventCreate(&b.ev1[i]));
      HMI_CUDA(cudaEventCreateWithFlags(&b.done[i], cudaEventDisableTiming));
    }
    const size_t lf = 4 * (d * d + d) + (d * f + f) + (f * d + d) + 4 * d;
    b.layers.resize(cfg->lower_layers);
    for (uint32_t l = 0; l < cfg->lower_layers; ++l) b.upload_layer(lower_f32 + l * lf, b.layers[l]);
    b.build_plans();
    HMI_CUDA(cudaDeviceSynchronize());
    *out = holder.release();
  });
}

int hmi_plot_builder_destroy(hmi_plot_builder* b) {
  return plot_guarded([&] { delete b; });
}

int hmi_plot_forward(hmi_plot_builder* b, uint32_t n, const uint32_t* key_len,
                     const uint32_t* keys, float* reps) {
  using namespace hmi_b200;
  return plot_guarded([&] {
    HMI_CHECK(b && (n == 0 || (key_len && keys && reps)), HMI_CONFIG_ERROR, "null argument");
    std::lock_guard<std::mutex> lock(b->impl.mu);
    HMI_CUDA(cudaSetDevice(b->impl.device));
    b->impl.forward(n, key_len, keys, reps);
  });
}

int hmi_plot_builder_stats(hmi_plot_builder* b, double* device_ms, uint64_t* rows) {
  using namespace hmi_b200;
  return plot_guarded([&] {
    HMI_CHECK(b != nullptr, HMI_CONFIG_ERROR, "null builder");
    std::lock_guard<std::mutex> lock(b->impl.mu);
    if (device_ms) *device_ms = b->impl.device_ms;
    if (rows) *rows = b->impl.rows_done;
  });
}

int hmi_plot_build_root(hmi_plot_builder* b, uint32_t n_seq, const uint32_t* seq_lens,
                        const uint32_t* tokens, hmi_plot_table** out) {
  using namespace hmi_b200;
  return plot_guarded([&] {
    HMI_CHECK(b && out && (n_seq == 0 || (seq_lens && tokens)), HMI_CONFIG_ERROR, "null argument");
    std::lock_guard<std::mutex> lock(b->impl.mu);
    HMI_CUDA(cudaSetDevice(b->impl.device));
    const CountMap sel = select_root(n_seq, seq_lens, tokens, b->impl.cfg.max_fragment,
                                     b->impl.cfg.vocab_size);
    *out = b->impl.materialize(sel);
  });
}

int hmi_plot_derive_branch(hmi_plot_builder* domain, const hmi_plot_table* root, uint32_t n_seq,
                           const uint32_t* seq_lens, const uint32_t* tokens, double alpha_percent,
                           hmi_plot_table** out) {
  using namespace hmi_b200;
  return plot_guarded([&] {
    HMI_CHECK(domain && root && out && (n_seq == 0 || (seq_lens && tokens)), HMI_CONFIG_ERROR,
              "null argument");
    HMI_CHECK(alpha_percent >= 0.0 && alpha_percent <= 100.0, HMI_CONFIG_ERROR,
              "alpha_percent must be in [0, 100]");
    HMI_CHECK(domain->impl.cfg.hidden_size == root->d && domain->impl.cfg.max_fragment == root->ngram,
              HMI_BUILD_ERROR, "domain model shape differs from the root table");
    std::lock_guard<std::mutex> lock(domain->impl.mu);
    HMI_CUDA(cudaSetDevice(domain->impl.device));
    const CountMap sel = select_branch(n_seq, seq_lens, tokens, root->ngram, alpha_percent);
    *out = domain->impl.materialize(sel);
  });
}

int hmi_plot_select_root(uint32_t ngram, uint32_t vocab, uint32_t n_seq, const uint32_t* seq_lens,
                         const uint32_t* tokens, hmi_plot_table** out) {
  using namespace hmi_b200;
  return plot_guarded([&] {
    HMI_CHECK(out && (n_seq == 0 || (seq_lens && tokens)), HMI_CONFIG_ERROR, "null argument");
    HMI_CHECK(ngram >= 1 && ngram <= kMaxFragment, HMI_CONFIG_ERROR, "ngram must be in [1, 5]");
    const CountMap sel = select_root(n_seq, seq_lens, tokens, ngram, vocab);
    auto* t = new hmi_plot_table;
    t->ngram = ngram;
    for (const auto& [key, fr] : sel) {
      t->key_len.push_back(static_cast<uint32_t>(key.size()));
      for (uint32_t i = 0; i < ngram; ++i) t->keys.push_back(i < key.size() ? key[i] : 0);
      t->freq.push_back(fr);
    }
    *out = t;
  });
}

int hmi_plot_select_branch(uint32_t ngram, uint32_t n_seq, const uint32_t* seq_lens,
                           const uint32_t* tokens, double alpha_percent, hmi_plot_table** out) {
  using namespace hmi_b200;
  return plot_guarded([&] {
    HMI_CHECK(out && (n_seq == 0 || (seq_lens && tokens)), HMI_CONFIG_ERROR, "null argument");
    HMI_CHECK(ngram >= 1 && ngram <= kMaxFragment, HMI_CONFIG_ERROR, "ngram must be in [1, 5]");
    const CountMap sel = select_branch(n_seq, seq_lens, tokens, ngram, alpha_percent);
    auto* t = new hmi_plot_table;
    t->ngram = ngram;
    for (const auto& [key, fr] : sel) {
      t->key_len.push_back(static_cast<uint32_t>(key.size()));
      for (uint32_t i = 0; i < ngram; ++i) t->keys.push_back(i < key.size() ? key[i] : 0);
      t->freq.push_back(fr);
    }
    *out = t;
  });
}

int hmi_plot_table_create(uint32_t ngram, uint32_t d, uint32_t n, const uint32_t* key_len,
                          const uint32_t* keys, const uint64_t* freq, const float* reps,
                          hmi_plot_table** out) {
  using namespace hmi_b200;
  return plot_guarded([&] {
    HMI_CHECK(out && (n == 0 || (key_len && keys)), HMI_CONFIG_ERROR, "null argument");
    HMI_CHECK(ngram >= 1 && ngram <= kMaxFragment, HMI_CONFIG_ERROR, "ngram must be in [1, 5]");
    auto* t = new hmi_plot_table;
    t->ngram = ngram;
    t->d = d;
    t->key_len.assign(key_len, key_len + n);
    t->keys.assign(keys, keys + static_cast<size_t>(n) * ngram);
    t->freq.assign(n, 1);
    if (freq) t->freq.assign(freq, freq + n);
    uint64_t rows = 0;
    for (uint32_t i = 0; i < n; ++i) {
      if (key_len[i] < 1 || key_len[i] > ngram) {
        delete t;
        throw HmiError(HMI_DIMENSION_ERROR, "key length must be in [1, ngram]");
      }
      rows += key_len[i];
    }
    if (reps) t->reps.assign(reps, reps + rows * d);
    *out = t;
  });
}

int hmi_plot_table_info(const hmi_plot_table* t, uint32_t* n_entries, uint64_t* n_rows,
                        uint32_t* has_reps) {
  return plot_guarded([&] {
    HMI_CHECK(t != nullptr, HMI_CONFIG_ERROR, "null table");
    uint64_t rows = 0;
    for (uint32_t l : t->key_len) rows += l;
    if (n_entries) *n_entries = static_cast<uint32_t>(t->key_len.size());
    if (n_rows) *n_rows = rows;
    if (has_reps) *has_reps = t->reps.empty() ? 0u : 1u;
  });
}

int hmi_plot_table_shape(const hmi_plot_table* t, uint32_t* ngram, uint32_t* d) {
  return plot_guarded([&] {
    HMI_CHECK(t != nullptr, HMI_CONFIG_ERROR, "null table");
    if (ngram) *ngram = t->ngram;
    if (d) *d = t->d;
  });
}

int hmi_plot_table_read(const hmi_plot_table* t, uint32_t* key_len, uint32_t* keys,
                        uint64_t* freq, float* reps) {
  return plot_guarded([&] {
    HMI_CHECK(t != nullptr, HMI_CONFIG_ERROR, "null table");
    if (key_len) std::copy(t->key_len.begin(), t->key_len.end(), key_len);
    if (keys) std::copy(t->keys.begin(), t->keys.end(), keys);
    if (freq) std::copy(t->freq.begin(), t->freq.end(), freq);
    if (reps) std::copy(t->reps.begin(), t->reps.end(), reps);
  });
}

int hmi_plot_table_free(hmi_plot_table* t) {
  return plot_guarded([&] { delete t; });
}

}  // extern "C"
