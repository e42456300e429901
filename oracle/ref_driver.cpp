// SPDX-License-Identifier: Apache-2.0
//
// ref_driver.cpp — TEST INFRASTRUCTURE ONLY.
//
// extern "C" driver over the *unmodified* reference library compiled from
// /root/reference/proj/src by oracle/build_ref.sh into oracle/_ref/libhmiref.so.
// It is the reference arm of bench.py (`--impl reference`) and the source of
// the golden fixtures in tests/golden/. Every computation is a call into the
// reference's own public API:
//   generate_model / generate_output_head   proj/src/transformer/weights.cpp:72-118
//   generate_adapter_set                    proj/src/adapters/adapter_set.cpp:15-25
//   build_root / derive_branch              proj/src/plot/table.cpp:29-104
//   VersionTree                             proj/src/plot/version_tree.cpp:11-107
//   resolve_window / retrieve_sequence      proj/src/plot/retrieval.cpp:23-124
//   higher_stack_forward / layer_forward    proj/src/transformer/model.cpp:84-185
//   DeviceSlotPool                          proj/src/adapters/device_pool.cpp:14-217
//   kernels::set_active                     proj/src/tensor/kernels.cpp:59-64
// The driver only converts flat arrays to the reference's types and back.
#include <atomic>
#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "hmi/adapters/adapter_set.hpp"
#include "hmi/adapters/device_pool.hpp"
#include "hmi/adapters/store.hpp"
#include "hmi/errors.hpp"
#include "hmi/plot/plot_io.hpp"
#include "hmi/plot/retrieval.hpp"
#include "hmi/plot/table.hpp"
#include "hmi/plot/version_tree.hpp"
#include "hmi/tensor/kernels.hpp"
#include "hmi/transformer/model.hpp"
#include "hmi/transformer/weights.hpp"

using namespace hmi;

namespace {
thread_local std::string g_err;

int fail(const std::exception& e, int code) {
  g_err = e.what();
  return code;
}

#define REF_TRY(...)                                              \
  try {                                                           \
    __VA_ARGS__;                                                       \
    return 0;                                                     \
  } catch (const DimensionError& e) { return fail(e, 1); }        \
  catch (const VocabularyError& e) { return fail(e, 2); }         \
  catch (const ConflictError& e) { return fail(e, 3); }           \
  catch (const CapacityError& e) { return fail(e, 4); }           \
  catch (const RoutingError& e) { return fail(e, 5); }            \
  catch (const ConfigError& e) { return fail(e, 6); }             \
  catch (const BuildError& e) { return fail(e, 7); }              \
  catch (const SchedulingBugError& e) { return fail(e, 8); }      \
  catch (const FormatError& e) { return fail(e, 9); }             \
  catch (const std::exception& e) { return fail(e, 99); }

struct RefConfig {
  uint32_t hidden_size, heads, lower_layers, higher_layers, ffn_size, vocab_size, mode,
      max_fragment, seed;
};

ModelConfig to_cfg(const RefConfig* c) {
  ModelConfig m;
  m.hidden_size = c->hidden_size;
  m.heads = c->heads;
  m.lower_layers = c->lower_layers;
  m.higher_layers = c->higher_layers;
  m.ffn_size = c->ffn_size;
  m.vocab_size = c->vocab_size;
  m.mode = static_cast<AttentionMode>(c->mode);
  m.max_fragment = c->max_fragment;
  m.seed = c->seed;
  return m;
}

void put(float*& out, const Matrix& m) {
  for (double v : m.flat()) *out++ = static_cast<float>(v);
}
void put(float*& out, const std::vector<double>& v) {
  for (double x : v) *out++ = static_cast<float>(x);
}

plot::PlotTable make_table(uint32_t ngram, uint32_t d, uint32_t n, const uint32_t* key_len,
                           const uint32_t* keys, const float* reps, const uint64_t* freq) {
  plot::PlotTable t;
  t.ngram = ngram;
  t.hidden_size = d;
  const float* r = reps;
  for (uint32_t e = 0; e < n; ++e) {
    plot::NGramKey key(keys + size_t(e) * ngram, keys + size_t(e) * ngram + key_len[e]);
    plot::PlotEntry entry;
    entry.freq = freq ? freq[e] : 1;
    entry.rep = Matrix(key_len[e], d);
    for (double& v : entry.rep.flat()) v = static_cast<double>(*r++);
    if (!t.entries.emplace(std::move(key), std::move(entry)).second) {
      throw FormatError("duplicate entry key", e);
    }
  }
  return t;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_set_kernels(const char* name) { return kernels::set_active(name) ? 0 : 6; }

const char* ref_active_kernels() { return kernels::active().name; }

// ---- model ------------------------------------------------------------------
void* ref_model_generate(const RefConfig* c) {
  try {
    return new ModelArtifacts(generate_model(to_cfg(c)));
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void ref_model_free(void* m) { delete static_cast<ModelArtifacts*>(m); }

// Higher-stack weights as f32 in HMI1 declaration order (model_io.cpp:19-36).
int ref_model_higher_f32(void* pm, float* out) {
  REF_TRY({
    const auto& m = *static_cast<ModelArtifacts*>(pm);
    for (const LayerWeights& l : m.higher) {
      put(out, l.wq); put(out, l.bq); put(out, l.wk); put(out, l.bk);
      put(out, l.wv); put(out, l.bv); put(out, l.wo); put(out, l.bo);
      put(out, l.w1); put(out, l.b1); put(out, l.w2); put(out, l.b2);
      put(out, l.ln1_gain); put(out, l.ln1_shift); put(out, l.ln2_gain); put(out, l.ln2_shift);
    }
  });
}

int ref_model_embeddings_f32(void* pm, float* tok, float* pos) {
  REF_TRY({
    const auto& m = *static_cast<ModelArtifacts*>(pm);
    put(tok, m.token_embedding);
    put(pos, m.position_embedding);
  });
}

int ref_model_save(void* pm, const char* path) {
  REF_TRY(save_model(*static_cast<ModelArtifacts*>(pm), path));
}

void* ref_model_load(const char* path) {
  try {
    return new ModelArtifacts(load_model(path));
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

// ---- adapters / heads -------------------------------------------------------
void* ref_adapter_generate(const char* task_id, const RefConfig* c, uint32_t r, uint64_t seed) {
  try {
    return new adapters::AdapterSet(adapters::generate_adapter_set(task_id, to_cfg(c), r, seed));
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void ref_adapter_free(void* s) { delete static_cast<adapters::AdapterSet*>(s); }

int ref_adapter_f32(void* ps, float* out) {
  REF_TRY({
    for (const AdapterParams& p : static_cast<adapters::AdapterSet*>(ps)->layers) {
      put(out, p.w_down); put(out, p.b_down); put(out, p.w_up); put(out, p.b_up);
    }
  });
}

int ref_adapter_save(void* ps, const char* path) {
  REF_TRY(adapters::save_adapter_set(*static_cast<adapters::AdapterSet*>(ps), path));
}

void* ref_head_generate(const char* task_id, uint32_t kind, uint32_t labels, const RefConfig* c,
                        uint64_t seed) {
  try {
    return new OutputHead(
        generate_output_head(task_id, static_cast<HeadKind>(kind), labels, to_cfg(c), seed));
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void ref_head_free(void* h) { delete static_cast<OutputHead*>(h); }

int ref_head_f32(void* ph, float* w, float* b) {
  REF_TRY({
    const auto& h = *static_cast<OutputHead*>(ph);
    put(w, h.w);
    put(b, h.b);
  });
}

// ---- PLOT tables / version tree ---------------------------------------------
void* ref_tree_create(uint32_t ngram, uint32_t d, uint32_t n, const uint32_t* key_len,
                      const uint32_t* keys, const float* reps, const uint64_t* freq) {
  try {
    return new plot::VersionTree(make_table(ngram, d, n, key_len, keys, reps, freq));
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void ref_tree_free(void* t) { delete static_cast<plot::VersionTree*>(t); }

// Returns the assigned version id (>= 1) or -code on error.
int64_t ref_tree_add_branch(void* pt, uint32_t parent_id, uint32_t n, const uint32_t* key_len,
                            const uint32_t* keys, const float* reps, const uint64_t* freq) {
  try {
    auto& tree = *static_cast<plot::VersionTree*>(pt);
    plot::PlotTable t =
        make_table(tree.root().ngram, tree.root().hidden_size, n, key_len, keys, reps, freq);
    t.parent_id = parent_id;
    return tree.add_branch(std::move(t));
  } catch (const RoutingError& e) {
    g_err = e.what();
    return -5;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -99;
  }
}

// Real build_root over a corpus (table.cpp:29-58): corpus given as n_seq
// sequences concatenated in `tokens` with lengths in `lens`.
void* ref_tree_build_root(void* pm, uint32_t n_seq, const uint32_t* lens, const uint32_t* tokens) {
  try {
    plot::Corpus corpus(n_seq);
    const uint32_t* t = tokens;
    for (uint32_t s = 0; s < n_seq; ++s) {
      corpus[s].assign(t, t + lens[s]);
      t += lens[s];
    }
    return new plot::VersionTree(plot::build_root(corpus, *static_cast<ModelArtifacts*>(pm)));
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

// derive_branch (table.cpp:60-104) from a domain corpus; returns version id.
int64_t ref_tree_derive_branch(void* pt, void* pm, uint32_t n_seq, const uint32_t* lens,
                               const uint32_t* tokens, double alpha) {
  try {
    auto& tree = *static_cast<plot::VersionTree*>(pt);
    plot::Corpus corpus(n_seq);
    const uint32_t* t = tokens;
    for (uint32_t s = 0; s < n_seq; ++s) {
      corpus[s].assign(t, t + lens[s]);
      t += lens[s];
    }
    return tree.add_branch(
        plot::derive_branch(tree.root(), corpus, *static_cast<ModelArtifacts*>(pm), alpha));
  } catch (const std::exception& e) {
    g_err = e.what();
    return -99;
  }
}

// Table export in std::map key order (the PLT1 order, plot_io.cpp:26-31).
int64_t ref_tree_table_size(void* pt, uint32_t version, uint64_t* rows) {
  const auto* t = static_cast<plot::VersionTree*>(pt)->version(version);
  if (!t) return -5;
  uint64_t r = 0;
  for (const auto& [k, e] : t->entries) r += k.size();
  if (rows) *rows = r;
  return static_cast<int64_t>(t->entries.size());
}

int ref_tree_table_export(void* pt, uint32_t version, uint32_t* key_len, uint32_t* keys,
                          float* reps, uint64_t* freq, uint32_t* parent) {
  REF_TRY({
    const auto* t = static_cast<plot::VersionTree*>(pt)->version(version);
    if (!t) throw RoutingError("no such version");
    if (parent) *parent = t->parent_id;
    size_t e = 0;
    for (const auto& [k, entry] : t->entries) {
      key_len[e] = static_cast<uint32_t>(k.size());
      for (uint32_t i = 0; i < t->ngram; ++i) keys[e * t->ngram + i] = i < k.size() ? k[i] : 0;
      if (freq) freq[e] = entry.freq;
      put(reps, entry.rep);
      ++e;
    }
  });
}

int ref_plot_persist(void* pt, uint32_t version, const char* path) {
  REF_TRY({
    const auto* t = static_cast<plot::VersionTree*>(pt)->version(version);
    if (!t) throw RoutingError("no such version");
    plot::persist(*t, path);
  });
}

// plot::load (plot_io.cpp:35-72) of a PLT1 file: hdr = {version, parent, ngram, d, count,
// alpha_centi}; arrays (nullable) in entry order, reps narrowed back to f32. Returns the
// reference's error class on failure (FormatError -> 9).
int ref_plt1_load(const char* path, uint32_t* hdr, uint32_t* key_len, uint32_t* keys, float* reps,
                  uint64_t* freq) {
  REF_TRY({
    const plot::PlotTable t = plot::load(path);
    hdr[0] = t.version_id;
    hdr[1] = t.parent_id;
    hdr[2] = t.ngram;
    hdr[3] = t.hidden_size;
    hdr[4] = static_cast<uint32_t>(t.entries.size());
    hdr[5] = t.alpha_centi;
    size_t e = 0;
    for (const auto& [k, entry] : t.entries) {
      if (key_len) key_len[e] = static_cast<uint32_t>(k.size());
      if (keys)
        for (uint32_t i = 0; i < t.ngram; ++i) keys[e * t.ngram + i] = i < k.size() ? k[i] : 0;
      if (freq) freq[e] = entry.freq;
      if (reps) put(reps, entry.rep);
      ++e;
    }
  });
}

// load_adapter_set / load_model status only (FormatError -> 9): the reference's verdict on a file
int ref_adp1_check(const char* path) { REF_TRY((void)adapters::load_adapter_set(path)); }
int ref_hmi1_check(const char* path) { REF_TRY((void)load_model(path)); }

// retrieve_sequence (retrieval.cpp:82-124) -> len x d doubles, plus the
// per-window resolve_window levels in the same sweep order (levels[p*n + k]
// for the k-th window covering p) for gather-index parity.
int ref_retrieve(void* pt, uint32_t version, const uint32_t* tokens, uint32_t len, uint32_t mode,
                 double* out, uint32_t* levels) {
  REF_TRY({
    const auto& tree = *static_cast<plot::VersionTree*>(pt);
    std::span<const uint32_t> toks(tokens, len);
    Matrix h = plot::retrieve_sequence(tree, version, toks, static_cast<AttentionMode>(mode));
    std::memcpy(out, h.data(), sizeof(double) * h.size());
    if (levels) {
      const uint32_t n = tree.root().ngram;
      std::fill(levels, levels + size_t(len) * n, 0u);
      if (mode == 1) {
        for (uint32_t i = 0; i < len; ++i) {
          const uint32_t start = i + 1 >= n ? i + 1 - n : 0;
          auto w = plot::resolve_window(tree, version, toks.subspan(start, i - start + 1));
          levels[size_t(i) * n] = w.levels[i - start];
        }
      } else {
        const uint32_t hl = (n - 1) / 2, hr = n - 1 - hl;
        std::vector<uint32_t> counts(len, 0);
        for (uint32_t c = 0; c < len; ++c) {
          const uint32_t start = c >= hl ? c - hl : 0;
          const uint32_t end = std::min(len - 1, c + hr);
          auto w = plot::resolve_window(tree, version, toks.subspan(start, end - start + 1));
          for (uint32_t p = start; p <= end; ++p) levels[size_t(p) * n + counts[p]++] = w.levels[p - start];
        }
      }
    }
  });
}

// ---- end-to-end reference path ----------------------------------------------
// For each request i: h = retrieve_sequence(tree, version[i], tokens_i) then
// higher_stack_forward(model, h, adapter layers of sets[i], *heads[i]).
// Runs `threads` host threads over disjoint request slices (compute is pure and
// read-shared). scores: n x max_labels; labels: n.
int ref_infer(void* pm, void* pt, uint32_t n, const uint32_t* version, void* const* sets,
              void* const* heads, const uint32_t* tokens, const uint32_t* lens, uint32_t stride,
              uint32_t max_labels, double* scores, int32_t* labels, int32_t* tags,
              uint32_t threads) {
  const auto& model = *static_cast<ModelArtifacts*>(pm);
  const auto& tree = *static_cast<plot::VersionTree*>(pt);
  std::atomic<uint32_t> next{0};
  std::atomic<int> status{0};
  auto work = [&]() {
    for (;;) {
      const uint32_t i = next.fetch_add(1);
      if (i >= n || status.load() != 0) return;
      try {
        std::span<const uint32_t> toks(tokens + size_t(i) * stride, lens[i]);
        Matrix h = plot::retrieve_sequence(tree, version[i], toks, model.config.mode);
        std::vector<const AdapterParams*> ad;
        if (sets && sets[i]) {
          for (const auto& p : static_cast<adapters::AdapterSet*>(sets[i])->layers) ad.push_back(&p);
        }
        HeadOutput o = higher_stack_forward(model, std::move(h), ad,
                                            *static_cast<OutputHead*>(heads[i]));
        for (size_t j = 0; j < o.scores.size() && j < max_labels; ++j)
          scores[size_t(i) * max_labels + j] = o.scores[j];
        labels[i] = o.label;
        if (tags) {
          for (size_t j = 0; j < o.tags.size(); ++j) tags[size_t(i) * stride + j] = o.tags[j];
        }
      } catch (const std::exception& e) {
        g_err = e.what();
        status.store(99);
      }
    }
  };
  if (threads <= 1) {
    work();
  } else {
    std::vector<std::thread> pool;
    for (uint32_t t = 0; t < threads; ++t) pool.emplace_back(work);
    for (auto& th : pool) th.join();
  }
  return status.load();
}

// ---- DeviceSlotPool trace replay (device_pool.cpp) ----------------------------
struct RefPool {
  adapters::AdapterStore store;
  std::unique_ptr<adapters::DeviceSlotPool> pool;
};

void* ref_pool_create(uint64_t capacity_bytes) {
  auto* p = new RefPool;
  p->pool = std::make_unique<adapters::DeviceSlotPool>(capacity_bytes);
  return p;
}

void ref_pool_free(void* p) { delete static_cast<RefPool*>(p); }

// Registers a task with `layers` layers of the given bottleneck (zero weights:
// only the byte accounting matters to the pool, adapter_set.hpp:24-27).
int ref_pool_register(void* pp, const char* task, uint32_t layers, uint32_t d, uint32_t r) {
  REF_TRY({
    adapters::AdapterSet s;
    s.task_id = task;
    for (uint32_t l = 0; l < layers; ++l) {
      AdapterParams a;
      a.layer_index = l;
      a.w_down = Matrix(d, r);
      a.b_down.assign(r, 0.0);
      a.w_up = Matrix(r, d);
      a.b_up.assign(d, 0.0);
      s.layers.push_back(std::move(a));
    }
    static_cast<RefPool*>(pp)->store.register_set(std::move(s));
  });
}

// op: 0 ensure_resident(all layers), 1 try_ensure_layer_resident(layer), 2 pin, 3 unpin,
//     4 touch, 5 evict(first id)
// Records per unique task: hit(0/1), bytes, and evicted names "a,b" (joined by ';' per record)
// Returns number of records, -1 if try_ensure returned nullopt, or -code.
int64_t ref_pool_op(void* pp, int op, uint32_t n_ids, const char* const* ids, uint32_t layer,
                    int32_t* hit, uint64_t* bytes, char* evicted, uint64_t evicted_cap) {
  auto* p = static_cast<RefPool*>(pp);
  try {
    std::vector<std::string> v(ids, ids + n_ids);
    std::vector<adapters::LoadRecord> recs;
    switch (op) {
      case 0: recs = p->pool->ensure_resident(p->store, v); break;
      case 1: {
        auto r = p->pool->try_ensure_layer_resident(p->store, v, layer);
        if (!r) return -1;
        recs = std::move(*r);
        break;
      }
      case 2: p->pool->pin(v); return 0;
      case 3: p->pool->unpin(v); return 0;
      case 4: p->pool->touch(v); return 0;
      case 5: return p->pool->evict(v.at(0)) ? 1 : 0;
      default: return -6;
    }
    std::string ev;
    for (size_t i = 0; i < recs.size(); ++i) {
      hit[i] = recs[i].hit ? 1 : 0;
      bytes[i] = recs[i].bytes;
      for (size_t j = 0; j < recs[i].evicted.size(); ++j) {
        if (j) ev += ",";
        ev += recs[i].evicted[j];
      }
      ev += ";";
    }
    if (evicted && evicted_cap) {
      std::strncpy(evicted, ev.c_str(), evicted_cap - 1);
      evicted[evicted_cap - 1] = 0;
    }
    return static_cast<int64_t>(recs.size());
  } catch (const CapacityError& e) {
    g_err = e.what();
    return -4;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -99;
  }
}

int ref_pool_stats(void* pp, uint64_t* out) {
  auto* p = static_cast<RefPool*>(pp)->pool.get();
  out[0] = p->hits();
  out[1] = p->loads();
  out[2] = p->resident_bytes();
  out[3] = p->max_resident_bytes_seen();
  out[4] = p->resident_task_count();
  return 0;
}

}  // extern "C"
