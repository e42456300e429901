// SPDX-License-Identifier: Apache-2.0
//
// hmi::sched::CudaBackend: see hmi/scheduler/cuda_backend.hpp. Compiled against the
// reference's public headers (proj/include) and linked by the host application together
// with the reference's own library and libhmi_b200.so.
#include "hmi/scheduler/cuda_backend.hpp"

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <utility>

#include "hmi_gpu.h"

namespace hmi::sched {

namespace {

// FormatError carries the byte offset where parsing stopped (errors.hpp:59-67); the ABI's
// message ends in "(offset N)".
std::size_t offset_of(const std::string& msg) {
  const auto at = msg.rfind("(offset ");
  if (at == std::string::npos) return 0;
  return static_cast<std::size_t>(std::strtoull(msg.c_str() + at + 8, nullptr, 10));
}

void check(int status) {
  if (status != HMI_OK) throw_on_status(status, hmi_gpu_last_error());
}

void put(std::vector<float>& out, const Matrix& m) {
  for (double v : m.flat()) out.push_back(static_cast<float>(v));
}

void put(std::vector<float>& out, const std::vector<double>& v) {
  for (double x : v) out.push_back(static_cast<float>(x));
}

}  // namespace

void throw_on_status(int status, const char* message) {
  const std::string msg = message ? message : "";
  switch (status) {
    case HMI_OK: return;
    case HMI_DIMENSION_ERROR: throw DimensionError(msg);
    case HMI_VOCABULARY_ERROR: throw VocabularyError(msg);
    case HMI_CONFLICT_ERROR: throw ConflictError(msg);
    case HMI_CAPACITY_ERROR: throw CapacityError(msg);
    case HMI_ROUTING_ERROR: throw RoutingError(msg);
    case HMI_CONFIG_ERROR: throw ConfigError(msg);
    case HMI_BUILD_ERROR: throw BuildError(msg);
    case HMI_SCHEDULING_BUG: throw SchedulingBugError(msg);
    case HMI_FORMAT_ERROR: throw FormatError(msg, offset_of(msg));
    default: throw std::runtime_error("CUDA backend status " + std::to_string(status) + ": " + msg);
  }
}

// ModelArtifacts -> the higher stack in the HMI1 per-layer order (model_io.cpp:19-36).
CudaBackend::CudaBackend(const ModelArtifacts& model, const CudaBackendConfig& config)
    : model_config_(model.config), config_(config) {
  model.config.validate();
  const ModelConfig& m = model.config;
  hmi_model_config c{m.hidden_size, m.heads, m.lower_layers, m.higher_layers, m.ffn_size,
                     m.vocab_size, static_cast<std::uint32_t>(m.mode), m.max_fragment, m.seed};
  if (model.higher.size() != m.higher_layers) throw DimensionError("model has no higher stack");
  std::vector<float> w;
  for (const LayerWeights& l : model.higher) {
    put(w, l.wq); put(w, l.bq); put(w, l.wk); put(w, l.bk); put(w, l.wv); put(w, l.bv);
    put(w, l.wo); put(w, l.bo); put(w, l.w1); put(w, l.b1); put(w, l.w2); put(w, l.b2);
    put(w, l.ln1_gain); put(w, l.ln1_shift); put(w, l.ln2_gain); put(w, l.ln2_shift);
  }
  hmi_gpu_options o{};
  o.precision = config.bf16 ? 1u : 0u;
  o.max_batch = config.max_batch_size;
  o.max_seq = config.max_seq;
  o.bottleneck = config.bottleneck;
  o.max_labels = config.max_labels;
  o.pipeline_mode = static_cast<std::uint32_t>(config.mode);
  o.pool_bytes = config.pool_capacity_bytes;
  o.max_tasks = config.max_tasks;
  o.max_instances = config.max_instances;
  o.max_heads = config.max_heads;
  o.max_versions = config.max_versions;
  o.max_new_tokens = config.max_new_tokens;
  check(hmi_gpu_create(config.device, &c, &o, w.data(), &ctx_));
}

CudaBackend::~CudaBackend() {
  if (ctx_) hmi_gpu_destroy(ctx_);
}

// ---- domain knowledge ------------------------------------------------------------------
void CudaBackend::add_table(const plot::PlotTable& t) {
  if (t.hidden_size != model_config_.hidden_size || t.ngram != model_config_.max_fragment) {
    throw DimensionError("PLOT table shape does not match the model");
  }
  std::vector<std::uint32_t> len, keys;
  std::vector<float> reps;
  len.reserve(t.entries.size());
  keys.reserve(t.entries.size() * t.ngram);
  for (const auto& [k, e] : t.entries) {  // std::map order: the PLT1 entry order
    len.push_back(static_cast<std::uint32_t>(k.size()));
    for (std::uint32_t i = 0; i < t.ngram; ++i) keys.push_back(i < k.size() ? k[i] : 0u);
    put(reps, e.rep);
  }
  check(hmi_gpu_upload_table(ctx_, t.version_id, t.parent_id,
                             static_cast<std::uint32_t>(len.size()), len.data(), keys.data(),
                             reps.data()));
  versions_[t.version_id] = true;
}

void CudaBackend::sync_tree(const plot::VersionTree& tree) {
  if (!versions_.count(tree.root().version_id)) add_table(tree.root());
  auto ids = tree.branch_ids();
  std::sort(ids.begin(), ids.end());  // parents are registered before their children
  for (std::uint32_t id : ids) {
    if (!versions_.count(id)) add_table(*tree.version(id));
  }
}

std::uint32_t CudaBackend::load_table(const std::filesystem::path& plt1) {
  std::uint32_t version = 0, parent = 0;
  check(hmi_gpu_upload_plt1(ctx_, plt1.c_str(), &version, &parent));
  versions_[version] = true;
  return version;
}

// ---- task knowledge --------------------------------------------------------------------
// AdapterSet -> the ADP1 body order (adapter_set.cpp:38-43): per layer w_down, b_down, w_up, b_up.
std::vector<float> CudaBackend::adapter_f32(const adapters::AdapterSet& s) const {
  if (s.layers.size() != model_config_.higher_layers) {
    throw DimensionError("adapter set must cover every higher layer");
  }
  std::vector<float> a;
  for (const AdapterParams& p : s.layers) {
    if (p.w_down.rows() != model_config_.hidden_size || p.bottleneck() != config_.bottleneck ||
        p.w_up.rows() != config_.bottleneck || p.w_up.cols() != model_config_.hidden_size) {
      throw DimensionError("adapter set " + s.task_id + " does not match d / bottleneck");
    }
    put(a, p.w_down); put(a, p.b_down); put(a, p.w_up); put(a, p.b_up);
  }
  return a;
}

void CudaBackend::register_set(const adapters::AdapterSet& set) {
  if (tasks_.count(set.task_id)) throw ConflictError("adapter set already registered: " + set.task_id);
  const std::vector<float> a = adapter_f32(set);
  std::uint32_t idx;
  if (!free_tasks_.empty()) {
    idx = free_tasks_.back();
  } else {
    if (next_task_ >= config_.max_tasks) throw CapacityError("max_tasks adapter sets registered");
    idx = next_task_;
  }
  check(hmi_gpu_register_task(ctx_, idx, a.data()));
  if (!free_tasks_.empty()) {
    free_tasks_.pop_back();
  } else {
    ++next_task_;
  }
  tasks_[set.task_id] = idx;
}

void CudaBackend::replace(const adapters::AdapterSet& set) {
  const std::vector<float> a = adapter_f32(set);
  check(hmi_gpu_replace_task(ctx_, task_index(set.task_id), a.data()));
}

void CudaBackend::erase(const std::string& task_id) {
  auto it = tasks_.find(task_id);
  if (it == tasks_.end()) return;  // AdapterStore::erase of an absent id is a no-op
  check(hmi_gpu_unregister_task(ctx_, it->second));
  free_tasks_.push_back(it->second);
  tasks_.erase(it);
}

void CudaBackend::sync_store(const adapters::AdapterStore& store) {
  auto ids = store.task_ids();
  std::sort(ids.begin(), ids.end());  // deterministic task indices
  for (const std::string& id : ids) {
    if (!tasks_.count(id)) register_set(*store.get(id));
  }
}

// ---- routing ---------------------------------------------------------------------------
void CudaBackend::bind_instance(const std::string& instance_id, const InstanceBinding& b) {
  if (instances_.count(instance_id)) throw ConflictError("instance already bound: " + instance_id);
  const std::uint32_t task = task_index(b.task_id);
  const OutputHead& h = b.head;
  if (h.w.rows() != model_config_.hidden_size || h.w.cols() != h.labels() || h.labels() == 0) {
    throw DimensionError("output head shape does not match the model");
  }
  auto hit = heads_.find(h.task_id);
  if (hit == heads_.end()) {
    const bool wide = h.kind == HeadKind::lm_logits && h.labels() > config_.max_labels;
    if (h.labels() > config_.max_labels && !wide) throw ConfigError("head labels exceed max_labels");
    if (next_head_ >= config_.max_heads) throw CapacityError("max_heads output heads registered");
    std::vector<float> w, bias;
    put(w, h.w);
    put(bias, h.b);
    check(hmi_gpu_register_head(ctx_, next_head_, static_cast<std::uint32_t>(h.kind),
                                static_cast<std::uint32_t>(h.labels()), w.data(), bias.data()));
    hit = heads_.emplace(h.task_id, HeadInfo{next_head_++, h.kind,
                                             static_cast<std::uint32_t>(h.labels()), wide}).first;
  } else if (hit->second.kind != h.kind || hit->second.labels != h.labels()) {
    throw ConflictError("a different output head is registered under " + h.task_id);
  }
  std::uint32_t idx;
  if (!free_instances_.empty()) {
    idx = free_instances_.back();
  } else {
    if (next_instance_ >= config_.max_instances) throw CapacityError("max_instances bound");
    idx = next_instance_;
  }
  check(hmi_gpu_bind_instance(ctx_, idx, b.version_id, task, hit->second.index));
  if (!free_instances_.empty()) {
    free_instances_.pop_back();
  } else {
    ++next_instance_;
  }
  instances_[instance_id] = idx;
  instance_head_[idx] = &hit->second;
}

void CudaBackend::unbind_instance(const std::string& instance_id) {
  auto it = instances_.find(instance_id);
  if (it == instances_.end()) return;
  check(hmi_gpu_unbind_instance(ctx_, it->second));
  instance_head_.erase(it->second);
  free_instances_.push_back(it->second);
  instances_.erase(it);
}

void CudaBackend::sync_instances(const InstanceTable& table) {
  std::vector<const std::pair<const std::string, InstanceBinding>*> todo;
  for (const auto& kv : table)
    if (!instances_.count(kv.first)) todo.push_back(&kv);
  std::sort(todo.begin(), todo.end(), [](auto* a, auto* b) { return a->first < b->first; });
  for (auto* kv : todo) bind_instance(kv->first, kv->second);
}

std::uint32_t CudaBackend::task_index(const std::string& task_id) const {
  auto it = tasks_.find(task_id);
  if (it == tasks_.end()) throw RoutingError("no adapter set registered for task " + task_id);
  return it->second;
}

std::uint32_t CudaBackend::instance_index(const std::string& instance_id) const {
  auto it = instances_.find(instance_id);
  if (it == instances_.end()) throw RoutingError("unknown instance " + instance_id);
  return it->second;
}

// ---- serving ---------------------------------------------------------------------------
CudaBackend::Packed CudaBackend::pack(const InferBatch& batch) const {
  Packed p;
  const std::size_t n = batch.requests.size();
  if (n == 0 || n > config_.max_batch_size) {
    throw DimensionError("batch size must be in [1, max_batch_size]");
  }
  for (const InferRequest& r : batch.requests) {
    if (r.tokens.empty()) throw DimensionError("request " + r.request_id + " has no tokens");
    p.stride = std::max<std::uint32_t>(p.stride, static_cast<std::uint32_t>(r.tokens.size()));
  }
  p.inst.resize(n);
  p.lens.resize(n);
  p.tokens.assign(n * p.stride, 0u);
  for (std::size_t i = 0; i < n; ++i) {
    const InferRequest& r = batch.requests[i];
    p.inst[i] = instance_index(r.instance_id);
    p.lens[i] = static_cast<std::uint32_t>(r.tokens.size());
    std::copy(r.tokens.begin(), r.tokens.end(), p.tokens.begin() + i * p.stride);
  }
  return p;
}

std::vector<HeadOutput> CudaBackend::unpack(const InferBatch& batch, const Packed& p,
                                            const std::vector<float>& scores,
                                            const std::vector<std::int32_t>& labels,
                                            const std::vector<std::int32_t>* tags) const {
  std::vector<HeadOutput> out(batch.requests.size());
  const std::size_t L = config_.max_labels;
  for (std::size_t i = 0; i < out.size(); ++i) {
    const HeadInfo& h = *instance_head_.at(p.inst[i]);
    HeadOutput& o = out[i];
    o.kind = h.kind;
    if (h.kind == HeadKind::token_tag) {  // rows [0, valid_len) (model.cpp:158-163)
      o.tags.assign(tags->begin() + i * p.stride, tags->begin() + i * p.stride + p.lens[i]);
      continue;
    }
    o.label = labels[i];
    if (h.wide) {
      o.scores = {static_cast<double>(scores[i * L])};
    } else {
      o.scores.assign(scores.begin() + i * L, scores.begin() + i * L + h.labels);
    }
  }
  return out;
}

std::vector<HeadOutput> CudaBackend::infer(const InferBatch& batch) {
  const Packed p = pack(batch);
  const std::uint32_t n = static_cast<std::uint32_t>(p.inst.size());
  std::vector<float> scores(static_cast<std::size_t>(n) * config_.max_labels);
  std::vector<std::int32_t> labels(n), tags(static_cast<std::size_t>(n) * p.stride);
  check(hmi_gpu_infer_batch(ctx_, n, p.inst.data(), p.tokens.data(), p.stride, p.lens.data(),
                            scores.data(), labels.data(), tags.data(), nullptr, 0, nullptr, 0,
                            nullptr));
  return unpack(batch, p, scores, labels, &tags);
}

std::vector<InferResult> CudaBackend::run(const std::vector<InferBatch>& batches, unsigned depth) {
  depth = std::clamp(depth, 1u, 4u);
  std::vector<InferResult> results;
  struct Pending {
    const InferBatch* batch;
    Packed p;
    std::uint64_t ticket;
  };
  std::deque<Pending> q;
  auto collect = [&]() {
    Pending& f = q.front();
    const std::uint32_t n = static_cast<std::uint32_t>(f.p.inst.size());
    std::vector<float> scores(static_cast<std::size_t>(n) * config_.max_labels);
    std::vector<std::int32_t> labels(n);
    check(hmi_gpu_wait_batch(ctx_, f.ticket, scores.data(), labels.data()));
    auto outs = unpack(*f.batch, f.p, scores, labels, nullptr);
    for (std::size_t i = 0; i < outs.size(); ++i) {
      InferResult r;
      r.request_id = f.batch->requests[i].request_id;
      r.batch_id = f.batch->batch_id;
      r.output = std::move(outs[i]);
      results.push_back(std::move(r));
    }
    q.pop_front();
  };
  for (const InferBatch& b : batches) {
    Pending f{&b, pack(b), 0};
    for (std::uint32_t k : f.p.inst) {
      if (instance_head_.at(k)->kind == HeadKind::token_tag) {
        // per-token tags are collected synchronously
        while (!q.empty()) collect();
        auto outs = infer(b);
        for (std::size_t i = 0; i < outs.size(); ++i) {
          InferResult r;
          r.request_id = b.requests[i].request_id;
          r.batch_id = b.batch_id;
          r.output = std::move(outs[i]);
          results.push_back(std::move(r));
        }
        f.batch = nullptr;
        break;
      }
    }
    if (!f.batch) continue;
    check(hmi_gpu_submit_batch(ctx_, static_cast<std::uint32_t>(f.p.inst.size()), f.p.inst.data(),
                               f.p.tokens.data(), f.p.stride, f.p.lens.data(), &f.ticket));
    q.push_back(std::move(f));
    if (q.size() >= depth) collect();
  }
  while (!q.empty()) collect();
  return results;
}

std::vector<std::vector<std::uint32_t>> CudaBackend::generate(const InferBatch& batch,
                                                              std::uint32_t n_new) {
  const Packed p = pack(batch);
  const std::uint32_t n = static_cast<std::uint32_t>(p.inst.size());
  std::vector<std::int32_t> toks(static_cast<std::size_t>(n) * n_new);
  check(hmi_gpu_generate(ctx_, n, p.inst.data(), p.tokens.data(), p.stride, p.lens.data(), n_new,
                         toks.data(), nullptr));
  std::vector<std::vector<std::uint32_t>> out(n);
  for (std::uint32_t i = 0; i < n; ++i)
    out[i].assign(toks.begin() + static_cast<std::size_t>(i) * n_new,
                  toks.begin() + static_cast<std::size_t>(i + 1) * n_new);
  return out;
}

}  // namespace hmi::sched
