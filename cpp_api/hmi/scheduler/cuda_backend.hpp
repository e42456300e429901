// SPDX-License-Identifier: Apache-2.0
//
// hmi::sched::CudaBackend — the reference-side binding of the B200 backend.
//
// The reference's scheduler runs each batch through a `Backend` of kind {numeric, simulated}
// whose stage_compute loops layer_forward per request.
// This is the third kind, `cuda`: it is compiled against the reference's own public headers
// (proj/include/hmi, unchanged) and forwards whole batches through this repo's C ABI
// (include/hmi_gpu.h, libhmi_b200.so). Callers keep the reference's types:
//
//   ModelArtifacts          weights.hpp:59-66        -> hmi_gpu_create (higher stack only)
//   plot::PlotTable /       table.hpp:26-40,         -> hmi_gpu_upload_table / _upload_plt1
//   plot::VersionTree       version_tree.hpp:30-57
//   adapters::AdapterSet /  adapter_set.hpp:15-31,   -> hmi_gpu_register_task / _replace_task /
//   adapters::AdapterStore  store.hpp:17-30             _unregister_task
//   InstanceBinding /       request.hpp:30-36        -> hmi_gpu_register_head / _bind_instance
//   InstanceTable
//   InferBatch -> HeadOutput request.hpp:22-25,       -> hmi_gpu_infer_batch (one call per batch)
//                            model.hpp:40-47             or _submit_batch / _wait_batch (run())
//
// String ids (task_id, instance_id, head task_id) map to dense indices here; the device only
// sees indices. Status codes come back as the reference's exception classes (errors.hpp:10-68),
// FormatError with its byte offset. One backend per GPU; like the reference's scheduler, one
// thread drives a backend, registrations apply between batches.
//
// Numerics: operands fp16 (bf16 with `bf16`), fp32 accumulate / LayerNorm / softmax, retrieval
// sums in f64; HeadOutput scores are the device's f32 logits widened to double. Tables are
// stored as PLT1 stores them (f32 reps): an in-memory build_root table (f64 reps,
// table.hpp:46-47) is quantised exactly as persist() would. A vocabulary-wide lm_logits head
// (labels > max_labels) reports its argmax token as `label` and scores = {its logit}.
#pragma once

#include <cstdint>
#include <filesystem>
#include <map>
#include <string>
#include <unordered_map>
#include <vector>

#include "hmi/adapters/store.hpp"
#include "hmi/errors.hpp"
#include "hmi/plot/version_tree.hpp"
#include "hmi/scheduler/request.hpp"
#include "hmi/transformer/model.hpp"

struct hmi_gpu_ctx;

namespace hmi::sched {

// SPEC.md:413-416 PipelineMode.
enum class PipelineMode : std::uint32_t { sync = 0, coarse = 1, fine = 2 };

struct CudaBackendConfig {
  int device = 0;
  std::uint32_t max_batch_size = 256;  // BatchQueue max_batch_size (request.hpp:50)
  std::uint32_t max_seq = 128;         // longest request; rows pad to a multiple of 128
  std::uint32_t bottleneck = 64;       // adapter r shared by every task (stack(), stacked.cpp:12-42)
  std::uint32_t max_labels = 8;        // widest cls / token_tag head
  PipelineMode mode = PipelineMode::fine;
  std::uint64_t pool_capacity_bytes = 0;  // DeviceSlotPool capacity, f32 accounting
                                          // (device_pool.hpp:40); 0 = every task resident
  std::uint32_t max_tasks = 1024, max_instances = 1024, max_heads = 1024, max_versions = 64;
  std::uint32_t max_new_tokens = 0;  // causal models: longest generate() continuation
  bool bf16 = false;                 // bf16 operands instead of fp16
};

// Throws the reference's exception class for an ABI status (no-op for HMI_OK).
void throw_on_status(int status, const char* message);

class CudaBackend {
 public:
  CudaBackend(const ModelArtifacts& model, const CudaBackendConfig& config);
  ~CudaBackend();
  CudaBackend(const CudaBackend&) = delete;
  CudaBackend& operator=(const CudaBackend&) = delete;

  // ---- domain knowledge (VersionTree)
  // One table version, under table.version_id / table.parent_id as the tree assigned them.
  void add_table(const plot::PlotTable& table);
  // The root and every branch of `tree` not uploaded yet (ascending version id).
  void sync_tree(const plot::VersionTree& tree);
  // A PLT1 file (plot_io.cpp:36-73), streamed straight to the device. Returns its version id.
  std::uint32_t load_table(const std::filesystem::path& plt1);

  // ---- task knowledge (AdapterStore)
  void register_set(const adapters::AdapterSet& set);  // ConflictError on duplicate
  void replace(const adapters::AdapterSet& set);       // RoutingError if absent
  void erase(const std::string& task_id);
  void sync_store(const adapters::AdapterStore& store);  // every set not registered yet

  // ---- routing (InstanceTable)
  // Binds instance -> (version, task adapters, head). Heads are deduplicated by head.task_id
  // (one hGPT vocabulary head shared by every instance is uploaded once); a different head
  // under a known head task_id is a ConflictError.
  void bind_instance(const std::string& instance_id, const InstanceBinding& binding);
  void unbind_instance(const std::string& instance_id);
  void sync_instances(const InstanceTable& table);

  // ---- serving
  // stage_retrieve + stage_prefetch + stage_compute + head for one batch,
  // outputs in request order. Unknown instance -> RoutingError; empty tokens -> DimensionError.
  std::vector<HeadOutput> infer(const InferBatch& batch);
  // run(queue) over formed batches with up to `depth` batches in flight
  // (submit / wait); results in batch order, then request order.
  std::vector<InferResult> run(const std::vector<InferBatch>& batches, unsigned depth = 2);
  // Greedy continuation of every request by n_new tokens (causal model, one wide lm head).
  std::vector<std::vector<std::uint32_t>> generate(const InferBatch& batch, std::uint32_t n_new);

  // ---- introspection
  std::uint32_t task_index(const std::string& task_id) const;          // RoutingError if unknown
  std::uint32_t instance_index(const std::string& instance_id) const;  // RoutingError if unknown
  hmi_gpu_ctx* context() const noexcept { return ctx_; }

 private:
  struct HeadInfo {
    std::uint32_t index;
    HeadKind kind;
    std::uint32_t labels;
    bool wide;
  };
  struct Packed {
    std::vector<std::uint32_t> inst, tokens, lens;
    std::uint32_t stride = 0;
  };
  Packed pack(const InferBatch& batch) const;
  std::vector<HeadOutput> unpack(const InferBatch& batch, const Packed& p,
                                 const std::vector<float>& scores,
                                 const std::vector<std::int32_t>& labels,
                                 const std::vector<std::int32_t>* tags) const;
  std::vector<float> adapter_f32(const adapters::AdapterSet& set) const;

  hmi_gpu_ctx* ctx_ = nullptr;
  ModelConfig model_config_;
  CudaBackendConfig config_;
  std::map<std::uint32_t, bool> versions_;
  std::unordered_map<std::string, std::uint32_t> tasks_, instances_;
  std::unordered_map<std::string, HeadInfo> heads_;
  std::unordered_map<std::uint32_t, const HeadInfo*> instance_head_;
  std::vector<std::uint32_t> free_tasks_, free_instances_;
  std::uint32_t next_task_ = 0, next_instance_ = 0, next_head_ = 0;
};

}  // namespace hmi::sched
