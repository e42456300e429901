// SPDX-License-Identifier: Apache-2.0
//
// A C++ caller holding the reference's own types drives the B200 backend through
// hmi::sched::CudaBackend (cpp_api/), and every HeadOutput is checked against the
// reference's own path on the same artefacts: higher_stack_forward(retrieve_sequence(...))
// (model.cpp:173-185, retrieval.cpp:82-124). The artefacts come from the
// reference's generators and builders (generate_model, build_root, derive_branch,
// generate_adapter_set, generate_output_head), linked from the reference library compiled
// by oracle/build_ref.sh — test infrastructure standing in for the application's own build.
//
//   test_cuda_backend --status-only   ABI status -> exception class mapping (no GPU)
//   test_cuda_backend [workdir]       everything (GPU)
//
// Prints one JSON summary line; exit code 0 iff every check passed.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <functional>
#include <random>
#include <string>
#include <vector>

#include "hmi/adapters/adapter_set.hpp"
#include "hmi/adapters/store.hpp"
#include "hmi/errors.hpp"
#include "hmi/plot/plot_io.hpp"
#include "hmi/plot/retrieval.hpp"
#include "hmi/plot/table.hpp"
#include "hmi/plot/version_tree.hpp"
#include "hmi/scheduler/cuda_backend.hpp"
#include "hmi/scheduler/request.hpp"
#include "hmi/tensor/kernels.hpp"
#include "hmi/transformer/model.hpp"
#include "hmi_gpu.h"

using namespace hmi;
namespace fs = std::filesystem;

static int failures = 0;
#define EXPECT(cond, what)                                                      \
  do {                                                                          \
    if (!(cond)) {                                                              \
      ++failures;                                                               \
      std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, what);       \
    }                                                                           \
  } while (0)

template <typename E>
static bool throws(const std::function<void()>& f, std::size_t* offset = nullptr) {
  try {
    f();
  } catch (const E& e) {
    if constexpr (std::is_same_v<E, FormatError>) {
      if (offset) *offset = e.offset();
    }
    return true;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "  unexpected exception: %s\n", e.what());
    return false;
  }
  return false;
}

static void status_mapping() {
  using sched::throw_on_status;
  EXPECT(throws<DimensionError>([] { throw_on_status(HMI_DIMENSION_ERROR, "d"); }), "DimensionError");
  EXPECT(throws<VocabularyError>([] { throw_on_status(HMI_VOCABULARY_ERROR, "v"); }), "VocabularyError");
  EXPECT(throws<ConflictError>([] { throw_on_status(HMI_CONFLICT_ERROR, "c"); }), "ConflictError");
  EXPECT(throws<CapacityError>([] { throw_on_status(HMI_CAPACITY_ERROR, "c"); }), "CapacityError");
  EXPECT(throws<RoutingError>([] { throw_on_status(HMI_ROUTING_ERROR, "r"); }), "RoutingError");
  EXPECT(throws<ConfigError>([] { throw_on_status(HMI_CONFIG_ERROR, "c"); }), "ConfigError");
  EXPECT(throws<BuildError>([] { throw_on_status(HMI_BUILD_ERROR, "b"); }), "BuildError");
  EXPECT(throws<SchedulingBugError>([] { throw_on_status(HMI_SCHEDULING_BUG, "s"); }),
         "SchedulingBugError");
  std::size_t off = 0;
  EXPECT(throws<FormatError>([] { throw_on_status(HMI_FORMAT_ERROR, "bad magic (offset 4)"); }, &off) &&
             off == 4,
         "FormatError carries the byte offset");
  EXPECT(throws<std::runtime_error>([] { throw_on_status(HMI_CUDA_ERROR, "cuda"); }), "CUDA error");
  bool ok = true;
  try {
    throw_on_status(HMI_OK, "");
  } catch (...) {
    ok = false;
  }
  EXPECT(ok, "HMI_OK does not throw");
}

// Token-window corpus over a vocabulary slice (Zipf-ish repetition so n-grams recur).
static plot::Corpus corpus(std::mt19937& rng, std::uint32_t lo, std::uint32_t hi, int seqs, int len) {
  plot::Corpus c;
  std::uniform_int_distribution<std::uint32_t> u(lo, hi - 1);
  std::uniform_int_distribution<int> rep(0, 3);
  for (int s = 0; s < seqs; ++s) {
    std::vector<std::uint32_t> seq;
    while (static_cast<int>(seq.size()) < len) {
      const std::uint32_t t = u(rng);
      seq.push_back(t);
      if (rep(rng) == 0 && seq.size() >= 3) {  // repeat a recent trigram
        const std::size_t k = seq.size() - 3;
        for (int j = 0; j < 3 && static_cast<int>(seq.size()) < len; ++j) seq.push_back(seq[k + j]);
      }
    }
    c.push_back(seq);
  }
  return c;
}

struct Ref {
  double err = 0.0;
  int label_agree = 0, labels = 0, tag_agree = 0, tags = 0;
};

int main(int argc, char** argv) {
  status_mapping();
  if (argc > 1 && std::strcmp(argv[1], "--status-only") == 0) {
    std::printf("{\"status_mapping\": %s}\n", failures ? "false" : "true");
    return failures ? 1 : 0;
  }
  const fs::path work = argc > 1 ? fs::path(argv[1]) : fs::temp_directory_path() / "hmi_cpp_backend";
  fs::create_directories(work);
  kernels::set_active("scalar");

  // ---- artefacts, built by the reference itself
  ModelConfig cfg;
  cfg.hidden_size = 256; cfg.heads = 4; cfg.lower_layers = 2; cfg.higher_layers = 2;
  cfg.ffn_size = 1024; cfg.vocab_size = 1024; cfg.mode = AttentionMode::encoder;
  cfg.max_fragment = 3; cfg.seed = 7;
  const ModelArtifacts model = generate_model(cfg);
  std::mt19937 rng(42);
  const plot::Corpus general = corpus(rng, 0, 1024, 4, 64);
  const plot::Corpus domain = corpus(rng, 100, 300, 8, 64);
  // persisted tables are float32-exact (plot_io.hpp:10-11): the device stores PLT1's f32 reps
  plot::persist(plot::build_root(general, model), work / "root.plt");
  plot::PlotTable root = plot::load(work / "root.plt");
  plot::VersionTree tree(root);
  plot::persist(plot::derive_branch(tree.root(), domain, model, 50.0), work / "branch.plt");
  const std::uint32_t branch = tree.add_branch(plot::load(work / "branch.plt"));

  const std::uint32_t r = 16, labels = 8;
  adapters::AdapterStore store;
  for (int t = 0; t < 6; ++t)
    store.register_set(adapters::generate_adapter_set("task" + std::to_string(t), cfg, r, 1000 + t));
  sched::InstanceTable table;
  for (int i = 0; i < 8; ++i) {
    sched::InstanceBinding b;
    b.version_id = i % 2 ? branch : 0;
    b.task_id = "task" + std::to_string(i % 6);
    const HeadKind kind = i == 6 ? HeadKind::token_tag : i == 7 ? HeadKind::lm_logits : HeadKind::cls_classify;
    b.head = generate_output_head("head" + std::to_string(i), kind, labels, cfg, 2000000 + i);
    table["inst" + std::to_string(i)] = b;
  }

  // ---- the backend, fed from the reference's registries
  sched::CudaBackendConfig bc;
  bc.max_batch_size = 16;
  bc.max_seq = 128;
  bc.bottleneck = r;
  bc.max_labels = labels;
  bc.max_tasks = 16; bc.max_instances = 16; bc.max_heads = 16; bc.max_versions = 8;
  sched::CudaBackend be(model, bc);
  be.sync_tree(tree);
  be.sync_store(store);
  be.sync_instances(table);

  auto make_batch = [&](std::size_t id, int n, unsigned seed) {
    sched::InferBatch b;
    b.batch_id = id;
    std::mt19937 g(seed);
    std::uniform_int_distribution<int> inst(0, 7), len(1, 128), src(0, 9);
    std::uniform_int_distribution<std::uint32_t> tok(0, cfg.vocab_size - 1);
    for (int k = 0; k < n; ++k) {
      sched::InferRequest q;
      q.request_id = "r" + std::to_string(id) + "_" + std::to_string(k);
      q.instance_id = "inst" + std::to_string(inst(g));
      const int L = k == 0 ? 128 : k == 1 ? 1 : k == 2 ? 2 : len(g);
      const auto& c = (src(g) < 5 ? domain : general)[g() % 4];
      for (int p = 0; p < L; ++p) q.tokens.push_back(src(g) == 0 ? tok(g) : c[p % c.size()]);
      b.requests.push_back(q);
    }
    return b;
  };

  // reference path per request: retrieve_sequence + higher_stack_forward
  auto reference = [&](const sched::InferRequest& q) {
    const sched::InstanceBinding& b = table.at(q.instance_id);
    const Matrix h0 = plot::retrieve_sequence(tree, b.version_id, q.tokens, cfg.mode);
    const auto set = store.get(b.task_id);
    std::vector<const AdapterParams*> ads;
    for (const auto& a : set->layers) ads.push_back(&a);
    return higher_stack_forward(model, h0, ads, b.head);
  };
  auto compare = [&](const sched::InferBatch& b, const std::vector<HeadOutput>& got, Ref& acc) {
    for (std::size_t i = 0; i < b.requests.size(); ++i) {
      const HeadOutput ref = reference(b.requests[i]);
      const HeadOutput& g = got[i];
      EXPECT(g.kind == ref.kind, "head kind");
      if (ref.kind == HeadKind::token_tag) {
        EXPECT(g.tags.size() == ref.tags.size() && g.label == -1, "token_tag shape");
        for (std::size_t p = 0; p < ref.tags.size() && p < g.tags.size(); ++p) {
          acc.tag_agree += g.tags[p] == ref.tags[p];
          ++acc.tags;
        }
        continue;
      }
      EXPECT(g.scores.size() == ref.scores.size(), "scores size");
      double mx = 0, dm = 0;
      for (std::size_t j = 0; j < ref.scores.size() && j < g.scores.size(); ++j) {
        mx = std::max(mx, std::fabs(ref.scores[j]));
        dm = std::max(dm, std::fabs(ref.scores[j] - g.scores[j]));
      }
      acc.err = std::max(acc.err, dm / mx);
      acc.label_agree += g.label == ref.label;
      ++acc.labels;
    }
  };

  Ref acc;
  std::vector<sched::InferBatch> batches;
  for (int k = 0; k < 3; ++k) batches.push_back(make_batch(k, 16, 7 + k));
  std::vector<std::vector<HeadOutput>> sync_out;
  for (const auto& b : batches) {
    sync_out.push_back(be.infer(b));
    compare(b, sync_out.back(), acc);
  }
  EXPECT(acc.err <= 2e-2, "logits within 2e-2 of the reference");
  EXPECT(acc.label_agree == acc.labels, "argmax labels equal the reference's");
  EXPECT(acc.tags > 0 && acc.tag_agree >= 0.99 * acc.tags, "token_tag agreement");

  // run(): the pipelined submit / wait path returns exactly what infer() returned
  const auto results = be.run(batches, 2);
  std::size_t k = 0;
  bool same = results.size() == 48;
  for (std::size_t bi = 0; bi < batches.size() && same; ++bi)
    for (std::size_t i = 0; i < batches[bi].requests.size(); ++i, ++k) {
      same &= results[k].request_id == batches[bi].requests[i].request_id &&
              results[k].batch_id == batches[bi].batch_id && results[k].output == sync_out[bi][i];
    }
  EXPECT(same, "run() equals infer() bit for bit, in batch order");

  // replace(): zero adapters are the identity -> the reference without adapters
  {
    adapters::AdapterSet zero = *store.get("task1");
    for (auto& l : zero.layers) {
      std::fill(l.w_down.flat().begin(), l.w_down.flat().end(), 0.0);
      std::fill(l.w_up.flat().begin(), l.w_up.flat().end(), 0.0);
      std::fill(l.b_down.begin(), l.b_down.end(), 0.0);
      std::fill(l.b_up.begin(), l.b_up.end(), 0.0);
    }
    be.replace(zero);
    store.replace(zero);
    sched::InferBatch b = make_batch(9, 4, 99);
    for (auto& q : b.requests) q.instance_id = "inst1";
    const auto got = be.infer(b);
    Ref z;
    compare(b, got, z);
    EXPECT(z.err <= 2e-2 && z.label_agree == z.labels, "replaced (zero) adapters");
  }

  // ---- error classes through the backend
  EXPECT(throws<ConflictError>([&] { be.register_set(*store.get("task2")); }), "duplicate set");
  EXPECT(throws<RoutingError>([&] {
           sched::InferBatch b = make_batch(20, 2, 5);
           b.requests[1].instance_id = "nobody";
           be.infer(b);
         }),
         "unknown instance");
  EXPECT(throws<VocabularyError>([&] {
           sched::InferBatch b = make_batch(21, 2, 6);
           b.requests[0].tokens[0] = cfg.vocab_size;
           be.infer(b);
         }),
         "token outside the vocabulary");
  EXPECT(throws<DimensionError>([&] {
           sched::InferBatch b = make_batch(22, 2, 7);
           b.requests[0].tokens.clear();
           be.infer(b);
         }),
         "empty request");
  EXPECT(throws<RoutingError>([&] {
           sched::InstanceBinding b = table.at("inst0");
           b.task_id = "absent";
           be.bind_instance("inst_new", b);
         }),
         "binding to an unknown task");
  EXPECT(throws<ConflictError>([&] { be.bind_instance("inst0", table.at("inst0")); }), "rebinding");
  EXPECT(throws<ConfigError>([&] { be.generate(make_batch(23, 2, 8), 2); }),
         "generation on an encoder model");
  {  // a truncated PLT1 file: FormatError with the offset where parsing stopped
    const fs::path bad = work / "bad.plt";
    fs::copy_file(work / "branch.plt", bad, fs::copy_options::overwrite_existing);
    fs::resize_file(bad, fs::file_size(bad) / 2);
    std::size_t off = 0;
    EXPECT(throws<FormatError>([&] { be.load_table(bad); }, &off) && off > 0,
           "truncated PLT1 -> FormatError(offset)");
    std::ofstream(work / "garbage.plt") << "not a table";
    EXPECT(throws<FormatError>([&] { be.load_table(work / "garbage.plt"); }), "bad magic");
  }
  {  // a pool holding one task's adapters cannot serve a batch needing two
    sched::CudaBackendConfig small = bc;
    small.pool_capacity_bytes = store.get("task0")->byte_size();
    sched::CudaBackend b2(model, small);
    b2.sync_tree(tree);
    b2.sync_store(store);
    b2.sync_instances(table);
    sched::InferBatch b = make_batch(30, 2, 11);
    b.requests[0].instance_id = "inst0";
    b.requests[1].instance_id = "inst2";
    EXPECT(throws<CapacityError>([&] { b2.infer(b); }), "working set above the pool capacity");
    b.requests[1].instance_id = "inst0";
    Ref c;
    compare(b, b2.infer(b), c);  // one task fits
    EXPECT(c.err <= 2e-2, "single-task batch through a one-task pool");
  }
  // erase + re-register under the same id gives the same outputs
  be.unbind_instance("inst3");
  be.erase("task3");
  EXPECT(throws<RoutingError>([&] { be.task_index("task3"); }), "erased task");
  be.register_set(*store.get("task3"));
  be.bind_instance("inst3", table.at("inst3"));
  {
    sched::InferBatch b = make_batch(40, 4, 13);
    for (auto& q : b.requests) q.instance_id = "inst3";
    Ref e;
    compare(b, be.infer(b), e);
    EXPECT(e.err <= 2e-2 && e.label_agree == e.labels, "erase + re-register");
  }

  std::printf(
      "{\"requests\": %d, \"max_rel_err\": %.3e, \"label_agree\": %d, \"labels\": %d, "
      "\"tag_agree\": %d, \"tags\": %d, \"run_equals_infer\": %s, \"failures\": %d}\n",
      acc.labels + 6, acc.err, acc.label_agree, acc.labels, acc.tag_agree, acc.tags,
      same ? "true" : "false", failures);
  return failures ? 1 : 0;
}
