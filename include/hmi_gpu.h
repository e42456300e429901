/* SPDX-License-Identifier: Apache-2.0
 *
 * hmi_gpu.h — C ABI of the B200-native batched multi-tenant hPLM forward pass.
 *
 * This is the drop-in boundary under the reference's C++ serving API. The
 * reference (proj/, C++20, CPU only) has no GPU backend; its SPEC defines a
 * scheduler `Backend` of kind {numeric, simulated} used by `stage_compute`
 * (SPEC.md:425-428, :461-469). This ABI is the third kind, `cuda`: the host
 * engine (paper_2504_17449_b200/host, or any C/C++/ctypes caller) registers
 * artefacts once and calls hmi_gpu_infer_batch() once per batch.
 *
 * Conventions
 *   - Plain pointers and sizes only; caller buffers are borrowed for the call.
 *   - Every entry point returns an int status (HMI_OK or an error class below).
 *     Status codes map 1:1 onto the reference's exception classes
 *     (proj/include/hmi/errors.hpp:10-68); hmi_gpu_last_error() returns the
 *     thread-local message. No exception crosses the ABI.
 *   - One context per GPU. hmi_gpu_infer_batch is not reentrant per context
 *     (one scheduler drains the queue); registration calls take a
 *     context mutex and apply between batches.
 *   - Float artefacts are passed exactly as stored in the reference's files:
 *     f32, row-major, declaration order (HMI1 model_io.cpp:19-36, ADP1
 *     adapter_set.cpp:38-43, PLT1 plot_io.cpp:17-33).
 */
#ifndef HMI_GPU_H_
#define HMI_GPU_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (errors.hpp:10-68) ------------------------------------ */
#define HMI_OK 0
#define HMI_DIMENSION_ERROR 1   /* DimensionError      errors.hpp:11  */
#define HMI_VOCABULARY_ERROR 2  /* VocabularyError     errors.hpp:17  */
#define HMI_CONFLICT_ERROR 3    /* ConflictError       errors.hpp:23  */
#define HMI_CAPACITY_ERROR 4    /* CapacityError       errors.hpp:29  */
#define HMI_ROUTING_ERROR 5     /* RoutingError        errors.hpp:35  */
#define HMI_CONFIG_ERROR 6      /* ConfigError         errors.hpp:40  */
#define HMI_BUILD_ERROR 7       /* BuildError          errors.hpp:46  */
#define HMI_SCHEDULING_BUG 8    /* SchedulingBugError  errors.hpp:53  */
#define HMI_FORMAT_ERROR 9      /* FormatError         errors.hpp:59  */
#define HMI_CUDA_ERROR 100      /* CUDA runtime / driver failure        */

/* Thread-local text of the last failing call on this thread. */
const char* hmi_gpu_last_error(void);

/* ---- configuration ------------------------------------------------------ */
/* ModelConfig (proj/include/hmi/transformer/config.hpp:10-24), HMI1 header order. */
typedef struct hmi_model_config {
  uint32_t hidden_size, heads, lower_layers, higher_layers, ffn_size, vocab_size;
  uint32_t mode; /* 0 encoder, 1 causal (AttentionMode) */
  uint32_t max_fragment;
  uint32_t seed;
} hmi_model_config;

/* Device-side options (not part of the reference; SURVEY.md §5 "device config"). */
typedef struct hmi_gpu_options {
  uint32_t precision;     /* GEMM/attention operand type: 0 fp16 (default), 1 bf16      */
  uint32_t max_batch;     /* max requests per batch (BatchQueue max_batch_size)          */
  uint32_t max_seq;       /* max request length; rows are padded to a multiple of 128    */
  uint32_t bottleneck;    /* adapter r shared by all tasks (stack() requires uniform r)  */
  uint32_t max_labels;    /* widest cls / token_tag / lm head                             */
  uint32_t pipeline_mode; /* 0 sync, 1 coarse, 2 fine                  */
  uint64_t pool_bytes;    /* DeviceSlotPool capacity in the reference's f32 byte
                             accounting (device_pool.hpp:40, adapter_set.hpp:24-27);
                             0 = room for every task (max_tasks)                          */
  uint32_t max_tasks, max_instances, max_heads, max_versions;
  uint32_t max_new_tokens; /* causal mode: longest hmi_gpu_generate continuation; > 0 keeps
                              every layer's prompt keys/values resident (KV cache)          */
  uint32_t reserved;
} hmi_gpu_options;

typedef struct hmi_gpu_ctx hmi_gpu_ctx;

/* Creates a context on `device` and uploads the shared higher-stack weights.
 * higher_f32: higher_layers blocks of the HMI1 per-layer payload, f32, in
 * declaration order wq,bq,wk,bk,wv,bv,wo,bo,w1,b1,w2,b2,ln1_gain,ln1_shift,
 * ln2_gain,ln2_shift (model_io.cpp:19-36; weights.hpp:15-21, matrices [in x out]).
 * Replaces: the numeric Backend's model artefacts.            */
int hmi_gpu_create(int device, const hmi_model_config* cfg, const hmi_gpu_options* opts,
                   const float* higher_f32, hmi_gpu_ctx** out);
int hmi_gpu_destroy(hmi_gpu_ctx* ctx);

/* ---- domain knowledge: PLOT version tree -------------------------------- */
/* Uploads one PLOT table version (PlotTable, plot/table.hpp:26-40; PLT1 body
 * plot_io.cpp:26-31). parent_id = 0xffffffff for the root. Entry e has key
 * key_len[e] tokens in keys[e*max_fragment ...] and key_len[e] rep rows in
 * reps (rows concatenated in entry order, hidden_size f32 each).
 * Errors mirror VersionTree::add_branch (version_tree.cpp:17-30) and PLT1 load
 * (plot_io.cpp:36-73): unknown parent -> ROUTING, duplicate version -> CONFLICT,
 * bad key length / duplicate key -> FORMAT, token >= vocab -> VOCABULARY.     */
int hmi_gpu_upload_table(hmi_gpu_ctx* ctx, uint32_t version_id, uint32_t parent_id,
                         uint32_t n_entries, const uint32_t* key_len, const uint32_t* keys,
                         const float* reps);

/* ---- task knowledge ------------------------------------------------------ */
/* Registers a task's adapter set (AdapterStore::register_set, store.cpp:9-18)
 * into pinned host memory; nothing is copied to HBM until a batch needs it.
 * adapter_f32: higher_layers blocks of w_down[d x r], b_down[r], w_up[r x d],
 * b_up[d] (the ADP1 body, adapter_set.cpp:38-43). Duplicate -> CONFLICT.    */
int hmi_gpu_register_task(hmi_gpu_ctx* ctx, uint32_t task_idx, const float* adapter_f32);
/* AdapterStore::replace (store.cpp:20-27): swaps the host copy; a resident
 * device copy is evicted so the next batch reloads it. Unknown -> ROUTING.   */
int hmi_gpu_replace_task(hmi_gpu_ctx* ctx, uint32_t task_idx, const float* adapter_f32);
/* AdapterStore::erase + DeviceSlotPool::evict (SPEC.md:527 delete_instance). */
int hmi_gpu_unregister_task(hmi_gpu_ctx* ctx, uint32_t task_idx);
/* Bulk register_set (start-up of 10,000 tenants): n tasks converted on `threads` host
 * threads (0 = the machine's cores, at most 32). All-or-nothing: any registered or repeated
 * index -> CONFLICT before any work; a failing task (by index order) is reported and
 * nothing is registered.                                                      */
int hmi_gpu_register_tasks(hmi_gpu_ctx* ctx, uint32_t n, const uint32_t* task_idx,
                           const float* const* adapter_f32, uint32_t threads);
/* Same from ADP1 files (adapter_set.cpp:48-75), read in parallel; a file whose header does
 * not match the model -> DIMENSION, a malformed one -> FORMAT.                           */
int hmi_gpu_register_task_files(hmi_gpu_ctx* ctx, uint32_t n, const uint32_t* task_idx,
                                const char* const* adp1_paths, uint32_t threads);

/* OutputHead (weights.hpp:45-53): kind 0 cls_classify, 1 token_tag,
 * 2 lm_logits; w [hidden x labels] f32, b [labels] f32.
 * An lm_logits head wider than max_labels (a vocabulary head, e.g. hGPT-2's
 * 50,257) is a "wide" head: its logits come from a tcgen05 GEMM over the
 * batch's final rows, the top-8 candidates are rescored in f64 from the f32
 * weights, and hmi_gpu_infer_batch reports label = argmax token and
 * scores[i*max_labels] = its logit (other columns 0). One wide head may be
 * shared by any number of instances; a batch may use at most one.           */
int hmi_gpu_register_head(hmi_gpu_ctx* ctx, uint32_t head_idx, uint32_t kind, uint32_t labels,
                          const float* w, const float* b);

/* InstanceBinding (scheduler/request.hpp:30-36) / VersionTree::bind_instance
 * (version_tree.cpp:81-93): instance -> (version, task, head).
 * Already bound -> CONFLICT; unknown version/task/head -> ROUTING.            */
int hmi_gpu_bind_instance(hmi_gpu_ctx* ctx, uint32_t instance_idx, uint32_t version_id,
                          uint32_t task_idx, uint32_t head_idx);
int hmi_gpu_unbind_instance(hmi_gpu_ctx* ctx, uint32_t instance_idx);

/* ---- serving ------------------------------------------------------------- */
/* One adapter load / hit of a batch, the LoadRecord of device_pool.hpp:27-33
 * (evicted task indices are written to the separate `evicted` array).        */
typedef struct hmi_load_record {
  uint32_t task;
  int32_t layer;          /* -1: all layers (ensure_resident), else the prefetched layer */
  int32_t hit;
  uint32_t n_evicted;
  uint64_t bytes;         /* reference f32 accounting */
  uint32_t evicted_offset;
  uint32_t pad;
} hmi_load_record;

/* Runs one mixed-tenant batch end to end (stage_compute for every higher layer,
 * SPEC.md:461-469, with on-device retrieval, routing, swap and head):
 *   instance_idx[n_req], tokens[n_req x stride] (request i uses lens[i] ids),
 *   scores[n_req x max_labels] f32 (cls / lm logits), labels[n_req] (argmax,
 *   -1 for token_tag), tags[n_req x stride] (token_tag only; nullable).
 * trace/evicted (nullable): up to trace_cap records / evicted_cap ids;
 * *n_trace receives the record count.                                           */
int hmi_gpu_infer_batch(hmi_gpu_ctx* ctx, uint32_t n_req, const uint32_t* instance_idx,
                        const uint32_t* tokens, uint32_t stride, const uint32_t* lens,
                        float* scores, int32_t* labels, int32_t* tags, hmi_load_record* trace,
                        uint32_t trace_cap, uint32_t* evicted, uint32_t evicted_cap,
                        uint32_t* n_trace);

/* Same batch with device-resident tokens/lens and device outputs; enqueued on
 * the context's compute stream without a host synchronisation (the routing
 * of instance_idx for the slot pool is host-side). d_tokens is [n_req x stride]. */
int hmi_gpu_infer_batch_device(hmi_gpu_ctx* ctx, uint32_t n_req, const uint32_t* instance_idx,
                               const uint32_t* d_tokens, uint32_t stride,
                               const uint32_t* d_lens, uint32_t max_len, float* d_scores,
                               int32_t* d_labels);
/* Greedy generation for causal (hGPT) models with a wide lm head: n_new
 * tokens per request, token k+1 = argmax lm_logits at the last row of the
 * prompt extended by tokens 1..k (apply_head, model.cpp:151-168; the reference
 * has no decode loop). The prompt runs as one batched forward
 * whose per-layer keys/values stay in HBM; each further token is one batched
 * single-row step per request (on-device causal retrieval of the new
 * position, cached attention, per-row tenant adapters). Every request must be
 * bound to the same wide lm head. out_tokens / out_logits: [n_req x n_new]
 * (out_logits nullable: the chosen token's f64-rescored logit).
 * Errors: n_new > max_new_tokens or encoder mode -> CONFIG.                  */
/* StageTrace: per (batch, stage, layer) intervals on three
 * logical workers on one clock (ms since hmi_gpu_trace(ctx, 1)): worker 0 cpu (the host's
 * submit: routing mirror, DeviceSlotPool decisions, staging), 1 io (the copy stream's adapter
 * H2D for one layer, stage 1 prefetch), 2 compute (stage 0 retrieve, stage 2 one layer's
 * compute, stage 3 head + result D2H). hmi_gpu_trace(ctx, 1) clears and starts recording;
 * hmi_gpu_stage_trace returns the records (n = total, at most cap written). */
typedef struct hmi_stage_record {
  uint64_t batch;
  uint32_t stage;  /* 0 retrieve, 1 prefetch, 2 compute, 3 head, 4 host submit */
  int32_t layer;   /* higher-stack layer, -1 none */
  uint32_t worker; /* 0 cpu, 1 io, 2 compute */
  uint32_t pad;
  double start_ms, end_ms;
} hmi_stage_record;
int hmi_gpu_trace(hmi_gpu_ctx* ctx, int enable);
int hmi_gpu_stage_trace(hmi_gpu_ctx* ctx, hmi_stage_record* out, uint32_t cap, uint32_t* n);

/* Asynchronous form of hmi_gpu_infer_batch for pipelined serving: the batch is enqueued
 * (inputs staged in pinned memory, H2D / compute / D2H on the context's streams) and a ticket
 * returned at once; hmi_gpu_wait_batch blocks until that batch finished and copies its
 * scores [n_req x max_labels] and labels out. At most 4 batches may be outstanding
 * (HMI_CAPACITY_ERROR beyond). Replaces nothing in the reference, whose scheduler drains
 * one batch at a time; it is how a serving loop overlaps batch k+1's host
 * work and copies with batch k's compute. */
int hmi_gpu_submit_batch(hmi_gpu_ctx* ctx, uint32_t n_req, const uint32_t* instance_idx,
                         const uint32_t* tokens, uint32_t stride, const uint32_t* lens,
                         uint64_t* ticket);
int hmi_gpu_wait_batch(hmi_gpu_ctx* ctx, uint64_t ticket, float* scores, int32_t* labels);

int hmi_gpu_generate(hmi_gpu_ctx* ctx, uint32_t n_req, const uint32_t* instance_idx,
                     const uint32_t* tokens, uint32_t stride, const uint32_t* lens,
                     uint32_t n_new, int32_t* out_tokens, float* out_logits);

/* Waits for every enqueued batch; returns the first device-side error. */
int hmi_gpu_synchronize(hmi_gpu_ctx* ctx);
/* cudaStream_t of the compute stream (for event timing by the caller). */
void* hmi_gpu_stream(hmi_gpu_ctx* ctx);

/* ---- introspection ------------------------------------------------------- */
/* Routing of the last batch: per request version/task/head, and the HBM slot
 * of each (request, layer) in slots[layer * n_req + i].                       */
int hmi_gpu_debug_routing(hmi_gpu_ctx* ctx, int32_t* version, int32_t* task, int32_t* head,
                          int32_t* slots);
/* Gather indices of the last batch: for row (i, p) and its k-th covering
 * window (ascending window order), the global PLOT rep row (upload order) and
 * the sub-gram level; -1 / 0 where unused. Arrays are [n_req x S x max_fragment]
 * with S = the batch's padded length (returned in *S).                        */
int hmi_gpu_debug_gather(hmi_gpu_ctx* ctx, int32_t* rows, int32_t* levels, uint32_t* S);
/* flags bit0: capture the f64 retrieval output h0 of the next batches;       */
/*       bit1: materialise the last layer's normalised rows (debug_hidden);   */
/*       bit2: decode steps as eager launches instead of the captured graph   */
/*             (the tests compare the two).                                   */
int hmi_gpu_set_debug(hmi_gpu_ctx* ctx, uint32_t flags);
int hmi_gpu_debug_h0(hmi_gpu_ctx* ctx, double* out);           /* [n_req x S x d] */
int hmi_gpu_debug_hidden(hmi_gpu_ctx* ctx, float* out);        /* final f32 rows */
/* DeviceSlotPool counters (device_pool.cpp:190-217):
 * out[0] hits, [1] loads, [2] resident_bytes, [3] max_resident_bytes_seen,
 * [4] resident_task_count, [5] capacity_bytes, [6] physical slots,
 * [7] bytes actually copied host->device (16-bit device layout).            */
int hmi_gpu_pool_stats(hmi_gpu_ctx* ctx, uint64_t* out);
int hmi_gpu_pool_slot(hmi_gpu_ctx* ctx, uint32_t task_idx, uint32_t layer, int32_t* slot);

/* Per-kernel-class device time (CUDA events around every launch while enabled). */
#define HMI_PROF_CLASSES 16
int hmi_gpu_profile(hmi_gpu_ctx* ctx, int enable);
/* ms[c], count[c] accumulated since enable; names in hmi_gpu_profile_name(c). */
int hmi_gpu_profile_read(hmi_gpu_ctx* ctx, double* ms, uint64_t* count);
const char* hmi_gpu_profile_name(int cls);

/* ---- seeded artefact generators (host only) ------------------------------ */
/* generate_model (weights.cpp:72-88): writes the f32 weights in HMI1 order;
 * any output pointer may be NULL (its draws are still consumed).              */
int hmi_generate_model(const hmi_model_config* cfg, float* token_embedding,
                       float* position_embedding, float* lower, float* higher);
/* generate_adapter_set (adapter_set.cpp:15-25): higher_layers ADP1 blocks.    */
int hmi_generate_adapter(const hmi_model_config* cfg, uint32_t bottleneck, uint64_t seed,
                         float* out);
/* generate_output_head (weights.cpp:105-118): w [d x labels], b [labels].    */
int hmi_generate_head(uint32_t hidden_size, uint32_t labels, uint64_t seed, float* w, float* b);

/* Engine counters: out[0] kernel launches, [1] batches, [2] host -> HBM adapter transfers
 * (one per run of consecutive slot images of a task),
 * [3] host NUMA node the pinned adapter store is bound to (UINT64_MAX: unknown). */
int hmi_gpu_counters(hmi_gpu_ctx* ctx, uint64_t* out);
/* Pinned-host (NUMA-local, as the adapter store) -> HBM copy rate on the copy stream:
 * `reps` copies of `bytes`; *gbps = GB/s. No reference counterpart (the reference's
 * transfer model is one PCIe link, device_pool.hpp:18-25); bench.py reports it per rank. */
int hmi_gpu_h2d_probe(hmi_gpu_ctx* ctx, uint64_t bytes, uint32_t reps, double* gbps);

/* ---- standalone slot-pool policy (host only; trace parity tests) ---------- */
typedef struct hmi_pool hmi_pool;
int hmi_pool_create(uint64_t capacity_bytes, hmi_pool** out);
int hmi_pool_destroy(hmi_pool* pool);
int hmi_pool_register(hmi_pool* pool, uint32_t task, uint32_t layers, uint64_t layer_bytes);
/* op 0 ensure_resident, 1 try_ensure_layer_resident(layer), 2 pin, 3 unpin, 4 touch,
 * 5 evict(tasks[0]). Returns records like hmi_gpu_infer_batch; *n_trace = -1
 * encodes try_ensure's nullopt. Errors as the reference (CAPACITY, ROUTING...). */
int hmi_pool_op(hmi_pool* pool, int op, uint32_t n, const uint32_t* tasks, uint32_t layer,
                hmi_load_record* trace, uint32_t trace_cap, uint32_t* evicted,
                uint32_t evicted_cap, int32_t* n_trace);
int hmi_pool_stats(hmi_pool* pool, uint64_t* out);
/* The same policy with the engine's physical placement: `physical_slots` slots in blocks of
 * `block_len` (a task's layer l goes to block * block_len + l of the block it claims; any free
 * slot when no block is free). Residency decisions are the byte budget's alone.
 * hmi_pool_slot: the slot of a resident (task, layer), else -1. */
int hmi_pool_create_placed(uint64_t capacity_bytes, uint32_t physical_slots, uint32_t block_len,
                           hmi_pool** out);
int hmi_pool_slot(hmi_pool* pool, uint32_t task, uint32_t layer, int32_t* slot);

/* ---- GPU PLOT builder --------------------------
 * The reference's offline table construction: build_root / derive_branch
 * (proj/src/plot/table.cpp:29-104) select keys exactly (std::map order, the PLT1
 * entry order; frequencies as the reference counts them) and each key's
 * representation is lower_stack_forward (proj/src/transformer/model.cpp:96-118),
 * computed on the GPU with the serving path's tcgen05 GEMM. A table can be handed
 * to hmi_gpu_upload_table as is (key_len, keys, reps).
 *   token_emb [vocab x d], pos_emb [max_fragment x d], lower_f32 = lower layers in
 *   the HMI1 per-layer order (as higher_f32 of hmi_gpu_create); max_rows bounds the
 *   rows per GPU pass (0: 16384). Errors: BUILD (empty corpus, no lower stack, domain
 *   model shape != root), CONFIG (alpha outside [0, 100]), DIMENSION (fragment length),
 *   VOCABULARY (token id).                                                    */
typedef struct hmi_plot_builder hmi_plot_builder;
typedef struct hmi_plot_table hmi_plot_table;
int hmi_plot_builder_create(int device, const hmi_model_config* cfg, const float* token_emb,
                            const float* pos_emb, const float* lower_f32, uint32_t precision,
                            uint32_t max_rows, hmi_plot_builder** out);
int hmi_plot_builder_destroy(hmi_plot_builder* b);
/* lower_stack_forward of n fragments (fragment i: key_len[i] tokens at keys[i * max_fragment]);
 * reps rows (sum key_len x d, f32) in fragment order */
int hmi_plot_forward(hmi_plot_builder* b, uint32_t n, const uint32_t* key_len,
                     const uint32_t* keys, float* reps);
/* device time (CUDA events around each GPU pass, H2D of keys to the last LayerNorm) and rows
 * computed since the builder was created */
int hmi_plot_builder_stats(hmi_plot_builder* b, double* device_ms, uint64_t* rows);
/* corpus = n_seq sequences of seq_lens[s] tokens, concatenated in `tokens` */
int hmi_plot_build_root(hmi_plot_builder* b, uint32_t n_seq, const uint32_t* seq_lens,
                        const uint32_t* tokens, hmi_plot_table** out);
int hmi_plot_derive_branch(hmi_plot_builder* domain_model, const hmi_plot_table* root,
                           uint32_t n_seq, const uint32_t* seq_lens, const uint32_t* tokens,
                           double alpha_percent, hmi_plot_table** out);
/* key selection only (no representations; host-only, no GPU needed) */
int hmi_plot_select_root(uint32_t ngram, uint32_t vocab, uint32_t n_seq, const uint32_t* seq_lens,
                         const uint32_t* tokens, hmi_plot_table** out);
int hmi_plot_select_branch(uint32_t ngram, uint32_t n_seq, const uint32_t* seq_lens,
                           const uint32_t* tokens, double alpha_percent, hmi_plot_table** out);
/* a table from arrays (e.g. a PLT1 body, plot_io.cpp:26-31); freq and reps nullable */
int hmi_plot_table_create(uint32_t ngram, uint32_t d, uint32_t n, const uint32_t* key_len,
                          const uint32_t* keys, const uint64_t* freq, const float* reps,
                          hmi_plot_table** out);
int hmi_plot_table_info(const hmi_plot_table* t, uint32_t* n_entries, uint64_t* n_rows,
                        uint32_t* has_reps);
int hmi_plot_table_shape(const hmi_plot_table* t, uint32_t* ngram, uint32_t* d);
/* key_len [n], keys [n x max_fragment] (zero padded), freq [n], reps [n_rows x d] (nullable) */
int hmi_plot_table_read(const hmi_plot_table* t, uint32_t* key_len, uint32_t* keys,
                        uint64_t* freq, float* reps);
int hmi_plot_table_free(hmi_plot_table* t);

/* ---- artefact ingest --------------------------
 * The reference's containers read straight into the f32 layouts above (no f64 round trip);
 * validation and FormatError cases as the reference readers (io/binary.cpp:62-123):
 *   PLT1 plot_io.cpp:17-72 · ADP1 adapter_set.cpp:27-75 · HMI1 model_io.cpp:83-115.
 * Two-phase reads: pass NULL arrays to get the sizes first.                 */
int hmi_plot_table_load(const char* path, hmi_plot_table** out, uint32_t* version_id,
                        uint32_t* parent_id, uint32_t* alpha_centi);
/* PLT1 writer (plot_io.cpp:17-33): entries in key order, reps f32 */
int hmi_plot_table_save(const hmi_plot_table* t, const char* path, uint32_t version_id,
                        uint32_t parent_id, const char* domain_label, uint32_t alpha_centi);
/* body = layers x (W_down [d x r], b_down [r], W_up [r x d], b_up [d]) f32, nullable */
int hmi_adapter_set_load(const char* path, char* task_id, uint32_t task_id_cap, uint32_t* layers,
                         uint32_t* d, uint32_t* r, float* body);
/* config, then (nullable) token_emb [vocab x d], pos_emb [max_fragment x d], lower / higher
 * layers in the HMI1 per-layer order */
int hmi_model_load(const char* path, hmi_model_config* cfg, float* token_emb, float* pos_emb,
                   float* lower_f32, float* higher_f32);
/* VersionTree::add_branch from a table handle (e.g. a loaded PLT1, or a GPU-built table) */
int hmi_gpu_upload_plot_table(hmi_gpu_ctx* ctx, uint32_t version_id, uint32_t parent_id,
                              const hmi_plot_table* t);
/* Streaming PLT1 ingest (plot_io.cpp:35-72): VersionTree::add_branch straight from a file.
 * Chunks are read into pinned memory and shipped whole; a kernel moves each entry's rep rows
 * into the reps arena while the host reads the next chunk (the host parses headers only).
 * Same checks and fail-closed commit as hmi_gpu_upload_table; ngram / d must match the model
 * (DIMENSION). *version_id / *parent_id (nullable) return the header's ids.                   */
int hmi_gpu_upload_plt1(hmi_gpu_ctx* ctx, const char* path, uint32_t* version_id,
                        uint32_t* parent_id);
/* AdapterStore::register_set from an ADP1 file (dimensions checked against the context) */
int hmi_gpu_register_task_file(hmi_gpu_ctx* ctx, uint32_t task_idx, const char* adp1_path);
int hmi_gpu_check_adapter_dims(hmi_gpu_ctx* ctx, uint32_t layers, uint32_t d, uint32_t r);

/* ---- peer rebalancing of tenants' adapters ---- */
/* A task migrating between shards (or a hot task replicated onto another GPU)
 * moves its HBM slots device to device over NVLink / NVSwitch instead of
 * re-crossing PCIe from the host store (DeviceSlotPool::ensure_resident,
 * device_pool.cpp:50-91, fed from a peer instead of AdapterStore::get). The
 * reference has one device and no such path; the numbers loaded are the ones
 * register_set would have loaded, bit for bit.                                */
#define HMI_EXPORT_MAX_LAYERS 64
typedef struct hmi_task_export {
  int32_t device;            /* CUDA ordinal of the source engine, in its process */
  int32_t pid;               /* source process id                                 */
  uint64_t arena;            /* source slot-arena device address (same process)   */
  uint8_t ipc_handle[64];    /* cudaIpcMemHandle_t of the arena (other processes) */
  uint64_t slot_bytes;       /* device bytes per (task, layer) slot               */
  uint64_t fingerprint;      /* d, layers, bottleneck, precision, slot layout     */
  uint32_t layers;
  uint32_t task_idx;
  int32_t slot[HMI_EXPORT_MAX_LAYERS]; /* per layer: physical slot in the arena   */
} hmi_task_export;
/* Makes every layer of a registered task resident in the source's slot pool
 * (under the LRU law, H2D for missing layers), pins it there until
 * hmi_gpu_release_export, and describes where its slots live.
 * Unknown task -> ROUTING; layers > HMI_EXPORT_MAX_LAYERS -> CONFIG.          */
int hmi_gpu_export_task(hmi_gpu_ctx* src, uint32_t task_idx, hmi_task_export* out);
/* Registers task_idx in dst and fills its slots from the exported ones by
 * peer copies (same process: direct; another process: CUDA IPC). The host
 * copy comes from adapter_f32 when given, else from the freshly filled HBM
 * slots (D2H, off any batch's critical path). Already registered -> CONFLICT;
 * model / bottleneck / precision mismatch -> CONFIG. *peer_bytes (nullable):
 * bytes moved device to device.                                               */
int hmi_gpu_import_task(hmi_gpu_ctx* dst, uint32_t task_idx, const hmi_task_export* ex,
                        const float* adapter_f32, uint64_t* peer_bytes);
/* Unpins an exported task; drop != 0 then unregisters it from the source
 * (a migration), drop == 0 keeps it (a replication of a hot tenant).         */
int hmi_gpu_release_export(hmi_gpu_ctx* src, uint32_t task_idx, int drop);

/* ---- standalone kernel probe (K1/K2 GEMM) ------------------------------ */
/* C[M x N] = epi(A[M x K] . B[g]^T + bias[g]) for a device-side tcgen05 GEMM,
 * host buffers in/out, used by the parity tests of the GEMM kernel alone.
 *   a16      : M*K 16-bit (fp16 or bf16 bits per `precision`)
 *   b16      : groups*N*K 16-bit, B stored [g][N][K] (i.e. W^T)
 *   bias     : groups*N f32
 *   tile_slot: M/128 ints selecting the group of each 128-row tile, or NULL
 *   res0/res1: optional M*N 16-bit residuals (epi flags 2/4)
 *   epi      : bit0 ReLU, bit1 +res0, bit2 +res0+res1, bit3 f32 output; probe flags:
 *              256 cta_group::2 pair kernel, 8192 no wave-tail split, 16384 the decode
 *              K-split cluster kernel (gemm_dec.cu)
 *   bn       : N-tile width (64, 128, 192 or 256); with 16384: (ks << 16) | width, or 0
 *              for the decode plan's own choice
 *   out      : M*N, 16-bit or f32 per epi bit3
 *   elapsed_ms (nullable): device time of one launch (CUDA events)        */
int hmi_gpu_gemm_probe(int device, int M, int N, int K, int groups, const uint16_t* a16,
                       const uint16_t* b16, const float* bias, const int32_t* tile_slot,
                       const uint16_t* res0, const uint16_t* res1, int epi, int bn,
                       int precision, void* out, float* elapsed_ms);

/* host -> HBM copy probe for adapter-slot transfers (n pieces of `bytes`): mode 0 one
 * contiguous copy, 1 n cudaMemcpyAsync, 3 zero-copy gather kernel over mapped pinned
 * memory with `ctas` CTAs; *gbps = achieved rate */
int hmi_gpu_copy_probe(int device, int n, size_t bytes, int mode, int ctas, double* gbps);

#ifdef __cplusplus
}
#endif

#endif /* HMI_GPU_H_ */
