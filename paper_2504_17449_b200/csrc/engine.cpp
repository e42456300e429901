// SPDX-License-Identifier: Apache-2.0
//
// The CUDA backend of the hPLM scheduler: one context per GPU.
//
// Restates, for a device, the SPEC's numeric Backend + stage_compute / run
// and the reference's per-request path it must equal
// (retrieve_sequence + higher_stack_forward):
//
//   host                     | copy stream               | compute stream
//   -------------------------+---------------------------+-------------------------------
//   route tasks (host mirror)|                           |
//   SlotPool decisions       | H2D adapter (task,layer)  | H2D tokens/lens/ids, slot deltas
//     (LRU/pin law of        |   -> HBM slot, per layer  | K6 route  (instance -> version,
//      DeviceSlotPool)       |   event ev_layer[l]       |            task, head, slots)
//                            |                           | K5 PLOT retrieval (Eq. 2/3)
//                            |                           | per layer l:
//                            |                           |   K1 QKV, K3 attention, K1 O
//                            |                           |   wait ev_layer[l]
//                            |                           |   K2 adapter down/up (+skip+res)
//                            |                           |   K4 LN1, K1 FFN1, K1 FFN2(+res)
//                            |                           |   K4 LN2
//                            |                           | K7 head + argmax, D2H
//
// Pipeline modes: sync waits for the previous batch and for
// every adapter copy before retrieval; coarse lets the next batch's copies run
// while the current batch computes (one event for all layers); fine waits per
// layer, so layer l+1's copies overlap layer l's compute.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <immintrin.h>
#include <sys/mman.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <fstream>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <set>
#include <string>
#include <thread>
#include <tuple>
#include <unordered_map>
#include <vector>

#include "decode.hpp"
#include "adapter.hpp"
#include "gemm.hpp"
#include "kernels.hpp"
#include "plot_builder.hpp"
#include "slot_pool.hpp"

namespace hmi_b200 {

void launch_apply_deltas(int32_t* table, const int32_t* pairs, int n, cudaStream_t stream);

namespace {

constexpr int kStaging = 4;
// StageTrace stages / workers (include/hmi_gpu.h hmi_stage_record)
constexpr int kStageRetrieve = 0, kStagePrefetch = 1, kStageCompute = 2, kStageHead = 3,
              kStageHost = 4;
constexpr int kWorkerCpu = 0, kWorkerIo = 1, kWorkerCompute = 2;

enum ProfClass {
  P_H2D = 0, P_ROUTE, P_RETRIEVE, P_QKV, P_ATTN, P_OPROJ, P_AD_DOWN, P_AD_UP, P_LN1, P_FFN1,
  P_FFN2, P_LN2, P_HEAD, P_D2H, P_COPY, P_STEP
};
const char* kProfNames[HMI_PROF_CLASSES] = {
    "h2d_inputs", "route",  "retrieve", "gemm_qkv", "attention", "gemm_oproj",
    "adapter_down", "adapter_up", "layernorm1", "gemm_ffn1", "gemm_ffn2", "layernorm2",
    "head", "d2h_outputs", "adapter_copy", "step"};

// Host f32 -> fp16 / bf16, round to nearest even. The F16C instruction and the bf16 bit
// rounding equal __float2half_rn / __float2bfloat16_rn on every non-NaN input (checked
// exhaustively over all 2^32 patterns) at a fraction of the software routines' cost.
__attribute__((target("f16c"))) static inline uint16_t f2h_f16c(float x) {
  return static_cast<uint16_t>(_cvtss_sh(x, _MM_FROUND_TO_NEAREST_INT));
}
static const bool kHasF16c = __builtin_cpu_supports("f16c");

uint16_t f2h(float x, int precision) {
  uint32_t u;
  std::memcpy(&u, &x, 4);
  const bool nan = (u & 0x7fffffffu) > 0x7f800000u;
  if (precision == 1) {
    if (!nan) return static_cast<uint16_t>((u + 0x7fffu + ((u >> 16) & 1u)) >> 16);
    __nv_bfloat16 b = __float2bfloat16_rn(x);
    return *reinterpret_cast<uint16_t*>(&b);
  }
  if (kHasF16c && !nan) return f2h_f16c(x);
  __half h = __float2half_rn(x);
  return *reinterpret_cast<uint16_t*>(&h);
}

template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  void alloc(size_t count) {
    free();
    if (count) HMI_CUDA(cudaMalloc(&p, count * sizeof(T)));
    n = count;
  }
  void free() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
};

struct LayerDev {
  void* mem = nullptr;  // one allocation per layer
  uint16_t *wqkv, *wo, *w1, *w2;  // [N][K] 16-bit (transposed from [in x out])
  float *bqkv, *bo, *b1, *b2, *ln1g, *ln1b, *ln2g, *ln2b;
  GemmPlan qkv, oproj, ad_down, ad_up, ffn1, ffn2;
  // LayerNorm folding (default mode): gamma folded into the consumer's weights, beta.W into
  // its bias, and the per-column sums of the folded 16-bit weights for the mean correction
  void* mem_fold = nullptr;
  uint16_t *wqkv_f = nullptr, *w1_f = nullptr;   // [N][K] 16-bit
  float *bqkv_f = nullptr, *cs_qkv = nullptr, *b1_f = nullptr, *cs_1 = nullptr;
};

// LN-fold of one consumer GEMM: W' = diag(gamma) W (rounded to 16-bit), b' = b + beta.W,
// colsum[n] = sum_k W'[k][n] over the rounded values (what the tensor core multiplies).
void fold_weights(const float* w, size_t in, size_t out, const float* bias, const float* gamma,
                  const float* beta, int prec, std::vector<uint16_t>& wt,
                  std::vector<float>& bias_f, std::vector<float>& colsum);

struct Staging {
  uint32_t* inst = nullptr;
  uint32_t* tokens = nullptr;
  int32_t* lens = nullptr;
  int32_t* delta = nullptr;  // (index, value) pairs
  float* scores = nullptr;
  int32_t* labels = nullptr;
  int32_t* tags = nullptr;
  int32_t* err = nullptr;
  cudaEvent_t done = nullptr;
  bool busy = false;
  // asynchronous submission (hmi_gpu_submit_batch): results held here until collected
  bool held = false;
  uint64_t ticket = 0;
  uint32_t n_req = 0;
};

struct Inflight {
  cudaEvent_t done;
  int staging;
  std::vector<uint32_t> tasks;
};

// N tile with the best (wave quantisation x per-tile efficiency); `pair`: units are 256-row
// CTA-pair tiles scheduled over sms/2 clusters (cta_group::2 kernel); `min_bn`: narrowest tile
// allowed. Per-tile efficiency of the pair kernel is measured (profiles/r01_gemm_sweep.txt:
// 256-wide pair tiles run 1.07-1.19x faster than 192-wide ones at equal wave counts; the
// 1-CTA kernel is less sensitive).
int pick_bn(int N, int m_tiles, int sms, bool pair = false, int min_bn = 64) {
  int best = -1;
  double best_eff = -1;
  if (pair) {
    m_tiles = (m_tiles + 1) / 2;
    sms /= 2;
  }
  for (int bn : {256, 192, 128, 64}) {
    if (N % bn || (pair && bn < 128) || bn < min_bn) continue;
    const long tiles = static_cast<long>(N / bn) * m_tiles;
    const long waves = (tiles + sms - 1) / sms;
    const double w = !pair ? 1.0 : bn == 256 ? 1.0 : bn == 192 ? 0.85 : 0.7;
    const double eff = w * static_cast<double>(tiles) / (waves * sms);
    if (eff > best_eff + 1e-9) {
      best_eff = eff;
      best = bn;
    }
  }
  return best;
}

void fold_weights(const float* w, size_t in, size_t out, const float* bias, const float* gamma,
                  const float* beta, int prec, std::vector<uint16_t>& wt,
                  std::vector<float>& bias_f, std::vector<float>& colsum) {
  wt.assign(in * out, 0);
  bias_f.assign(out, 0.f);
  colsum.assign(out, 0.f);
  for (size_t o = 0; o < out; ++o) {
    double cs = 0.0, bb = static_cast<double>(bias[o]);
    for (size_t i = 0; i < in; ++i) {
      const float wv = w[i * out + o];
      const uint16_t h = f2h(static_cast<float>(static_cast<double>(gamma[i]) * wv), prec);
      wt[o * in + i] = h;
      float back;
      if (prec == 1) {
        const uint32_t u = static_cast<uint32_t>(h) << 16;
        std::memcpy(&back, &u, 4);
      } else {
        back = __half2float(*reinterpret_cast<const __half*>(&h));
      }
      cs += back;
      bb += static_cast<double>(beta[i]) * wv;
    }
    colsum[o] = static_cast<float>(cs);
    bias_f[o] = static_cast<float>(bb);
  }
}

}  // namespace

// Pinned adapter store placed on the GPU's own NUMA node: on a two-socket 8-GPU box the
// adapter misses then cross PCIe only, not the socket link as well. Pages are mmap'd, bound
// with mbind(MPOL_PREFERRED, node) (falls back to other nodes when that one is full), faulted
// in, then page-locked with cudaHostRegister (portable: any device may copy from them).
static int gpu_numa_node(int device) {
  char bus[64] = {};
  if (cudaDeviceGetPCIBusId(bus, sizeof bus, device) != cudaSuccess) return -1;
  std::string id(bus);
  for (auto& ch : id) ch = static_cast<char>(std::tolower(static_cast<unsigned char>(ch)));
  for (const std::string& cand : {id, id.size() > 4 && id.rfind("0000", 0) == 0 ? id.substr(4) : id}) {
    std::ifstream in("/sys/bus/pci/devices/" + cand + "/numa_node");
    int node = -1;
    if (in >> node) return node;
  }
  return -1;
}

static uint8_t* host_alloc_local(size_t bytes, int node) {
  void* p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
  HMI_CHECK(p != MAP_FAILED, HMI_CAPACITY_ERROR, "pinned adapter store: mmap failed");
  if (node >= 0 && node < 64) {
    const unsigned long mask = 1ul << node;
    constexpr int kMpolPreferred = 1;
    syscall(SYS_mbind, p, bytes, kMpolPreferred, &mask, 64ul, 0u);  // best effort
  }
  std::memset(p, 0, bytes);  // fault the pages in under the policy
  const cudaError_t e = cudaHostRegister(p, bytes, cudaHostRegisterPortable);
  if (e != cudaSuccess) {
    munmap(p, bytes);
    HMI_CUDA(e);
  }
  return static_cast<uint8_t*>(p);
}

static void host_free_local(uint8_t* p, size_t bytes) {
  cudaHostUnregister(p);
  munmap(p, bytes);
}

struct Ctx {
  int device = 0;
  hmi_model_config cfg{};
  hmi_gpu_options opt{};
  int d = 0, f = 0, L = 0, heads = 0, ngram = 3, r = 0, r_pad = 0;
  int S_max = 0, max_rows = 0, tile_stride = 0;
  size_t slot_bytes = 0;         // device bytes per (task, layer)
  uint64_t ref_layer_bytes = 0;  // reference f32 accounting per layer
  cudaStream_t compute = nullptr, copy = nullptr;
  std::mutex mu;

  std::vector<LayerDev> layers;
  std::vector<AttnPlan> attn;  // per layer when the prompt KV cache is kept, else one
  // activations
  DevBuf<uint16_t> h16, qkv16, ctx16, a16, mid16, x16, ffn16;
  DevBuf<float> y32, h32;
  DevBuf<double> h64;
  // per-batch device inputs / routing
  DevBuf<uint32_t> d_inst, d_tokens;
  DevBuf<int32_t> d_lens, d_delta, d_req_version, d_req_task, d_req_head, d_tile_slot, d_err;
  DevBuf<int32_t> d_gather, d_levels;
  DevBuf<float> d_scores;
  DevBuf<int32_t> d_labels, d_tags;
  // tables
  DevBuf<int32_t> d_inst_version, d_inst_task, d_inst_head, d_slot_of;
  std::vector<int32_t> h_inst_version, h_inst_task, h_inst_head;
  // PLOT
  std::vector<PlotSlot> h_slots;
  uint64_t n_keys = 0;
  std::vector<int32_t> h_parent;  // -2 = absent
  DevBuf<PlotSlot> d_slots;
  DevBuf<int32_t> d_parent;
  DevBuf<float> d_reps;
  uint64_t rep_rows = 0;
  // heads
  DevBuf<float> d_head_arena;
  uint64_t head_floats = 0;
  DevBuf<int64_t> d_head_off;
  DevBuf<int32_t> d_head_labels, d_head_kind;
  std::vector<int64_t> h_head_off;
  std::vector<int32_t> h_head_labels, h_head_kind;
  // adapters: pinned host store + HBM slot arena
  std::unique_ptr<SlotPool> pool;
  DevBuf<uint8_t> arena;
  std::vector<uint8_t*> store;  // per task, L * slot_bytes pinned, or null
  std::vector<std::pair<uint8_t*, size_t>> pinned_chunks;  // mmap'd + cudaHostRegister'ed
  int numa_node = -1;  // host NUMA node of the GPU's PCIe root (sysfs), -1 if unknown
  std::vector<uint8_t*> free_blocks;
  uint8_t* chunk_cur = nullptr;
  size_t chunk_left = 0;
  uint64_t bytes_copied = 0;
  uint64_t n_launches = 0, n_batches = 0, n_copies = 0;
  uint64_t next_ticket = 0;
  std::vector<cudaEvent_t> ev_layer;
  struct CopyItem {
    uint32_t task, layer;
    int32_t slot;
  };
  std::vector<CopyItem> copy_items;
  // a second copy stream: consecutive runs alternate between two DMA queues so one run's
  // setup overlaps the other's transfer; it joins `copy` before the layers' events
  cudaStream_t copy2 = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // fine mode: d_ready[l] = sequence number of the last batch whose layer-l adapter copies are
  // complete, written by the copy stream (cuStreamWriteValue32); the fused adapter kernel waits
  // on it on the device, so the compute stream carries no cross-stream event wait
  DevBuf<uint32_t> d_ready;
  StreamWriteValue32Fn write_value32 = nullptr;
  uint32_t ready_seq = 0;
  // decode step captured once per (batch shape, head, tables) and replayed with cudaGraphLaunch
  // (debug flag 4: eager launches every step)
  std::map<std::tuple<int, int, int, uint64_t>, cudaGraphExec_t> dec_graphs;
  uint64_t tables_epoch = 0;
  // A captured decode graph holds raw pointers into the reps arena, the head arena, the lm
  // logits buffer and the lm GEMM plans' tensor maps: anything that reallocates one of them
  // drops every graph first (they are recaptured on the next generate).
  void drop_decode_graphs() {
    if (dec_graphs.empty()) return;
    HMI_CUDA(cudaStreamSynchronize(compute));
    for (auto& [k, g] : dec_graphs) cudaGraphExecDestroy(g);
    dec_graphs.clear();
    ++tables_epoch;
  }

  // peer rebalancing: export pins per task, peer arenas opened over CUDA IPC, bytes moved
  std::map<uint32_t, int> exported;
  std::map<std::string, void*> ipc_open;
  int ipc_state = 0;  // 0 not asked yet, 1 handle valid, -1 arena not exportable
  cudaIpcMemHandle_t ipc_handle{};
  uint64_t peer_bytes = 0;
  uint64_t fingerprint() const {
    uint64_t h = 0xcbf29ce484222325ULL;
    for (uint64_t v : {uint64_t(d), uint64_t(L), uint64_t(r), uint64_t(r_pad), uint64_t(opt.precision),
                       uint64_t(slot_bytes)}) {
      for (int i = 0; i < 8; ++i) h = (h ^ ((v >> (8 * i)) & 0xff)) * 0x100000001b3ULL;
    }
    return h;
  }
  // staging / in-flight batches
  Staging stg[kStaging];
  int stg_next = 0;
  std::deque<Inflight> inflight;
  int sticky_err = 0;  // first device-side error of a batch retired without a waiter
  void raise_sticky() {
    const int e = sticky_err;
    sticky_err = 0;
    if (e) throw HmiError(e, "device-side error in an earlier batch (status " + std::to_string(e) + ")");
  }
  // last batch (introspection)
  uint32_t last_n = 0, last_S = 0;
  uint32_t debug_flags = 0;
  // adapter up projection as tenant K blocks of the O projection (kEpiExt) when r <= 64 and
  // d % 128 == 0, else a separate tenant-grouped up GEMM (+ skip + residual)
  bool oproj_ext = true;
  // adapter fold (adapter.cu): the layers' f32 Wo / bo, and device staging for slot images
  DevBuf<float> wo32, bo32;
  DevBuf<uint8_t> fold_in, fold_out;
  size_t fold_cap = 0;  // tasks per staging pass
  cudaStream_t fold_stream = nullptr;
  DevBuf<float2> d_stats1, d_stats2;  // partial row (sum, sumsq) of y1 / y2, [rows][kStatsLd]
  static constexpr int kStatsLd = kStatsStride;
  int stats1_bn = 0, stats2_bn = 0, stats1_n = 0, stats2_n = 0;
  // causal generation: each layer's prompt q|k|v stays in qkv16 (KV cache); the generated
  // rows' k|v go to kv_tail [L][max_batch][max_new][2d]
  bool kv = false;
  int Bp = 0;  // max_batch rounded up to 128 (rows of the single-row decode GEMMs)
  DevBuf<uint16_t> qkv_dec, kv_tail, hdec16;
  DevBuf<float> hdec32, lm_logits;
  DevBuf<uint32_t> gen_tokens;
  DevBuf<int32_t> gen_pos, gen_out;
  DevBuf<float> gen_logit;
  int gen_stride = 0;
  struct DecPlans {
    GemmPlan qkv, oproj, ffn1, ffn2;
    // K-split cluster GEMMs (gemm_dec.cu); fn == nullptr: no (tile, split) fits this shape and
    // the persistent K1 plan above runs instead
    DecGemmPlan kqkv, koproj, kffn1, kffn2;
    AttnDecodeMaps attn;  // TMA maps over this layer's prompt q|k|v and generated k|v
  };
  std::vector<DecPlans> dec;
  // wide lm heads (kind 2, labels > max_labels): 16-bit [V_pad][d] GEMM operand + padded bias
  struct LmHead {
    int V = 0, V_pad = 0;
    uint16_t* w16 = nullptr;
    float* bias = nullptr;
    float* wT = nullptr;  // [V][d] f32: the exact weights per candidate column, contiguous
    GemmPlan plan;
  };
  std::map<int, LmHead> lm_heads;
  uint16_t* qkv_at(int l) const {
    return qkv16.p + (kv ? static_cast<size_t>(l) * max_rows * 3 * d : 0);
  }
  void build_lm_plan(LmHead& h);
  // profiling
  bool prof = false;
  // StageTrace: per (batch, stage, layer) intervals on three logical
  // workers, cpu (host submit), io (copy stream), compute (compute stream), one clock whose
  // origin is `trace_epoch` (recorded on an idle device when tracing is enabled)
  struct TraceEv {
    uint64_t batch;
    int stage, layer, worker;
    cudaEvent_t a = nullptr, b = nullptr;
    double host_a = 0, host_b = 0;
  };
  bool trace_on = false;
  cudaEvent_t trace_epoch = nullptr;
  std::chrono::steady_clock::time_point trace_host0;
  std::vector<TraceEv> trace_evs;
  double host_ms() const {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - trace_host0)
        .count();
  }
  // brackets the work `fn` enqueues on `stream` with a traced interval
  template <typename F>
  void traced(int stage, int layer, int worker, cudaStream_t stream, F&& fn) {
    if (!trace_on) {
      fn();
      return;
    }
    TraceEv e{n_batches, stage, layer, worker};
    HMI_CUDA(cudaEventCreate(&e.a));
    HMI_CUDA(cudaEventCreate(&e.b));
    HMI_CUDA(cudaEventRecord(e.a, stream));
    fn();
    HMI_CUDA(cudaEventRecord(e.b, stream));
    trace_evs.push_back(e);
  }
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> prof_pending;
  std::vector<cudaEvent_t> prof_free;
  double prof_ms[HMI_PROF_CLASSES] = {};
  uint64_t prof_cnt[HMI_PROF_CLASSES] = {};

  ~Ctx();

  cudaEvent_t ev() {
    cudaEvent_t e;
    if (!prof_free.empty()) {
      e = prof_free.back();
      prof_free.pop_back();
    } else {
      HMI_CUDA(cudaEventCreate(&e));
    }
    return e;
  }
  template <typename F>
  void timed(int cls, cudaStream_t s, F&& fn) {
    if (!prof) {
      fn();
      return;
    }
    cudaEvent_t a = ev(), b = ev();
    HMI_CUDA(cudaEventRecord(a, s));
    fn();
    HMI_CUDA(cudaEventRecord(b, s));
    prof_pending.push_back({cls, {a, b}});
  }
  void prof_collect() {
    for (auto& [cls, e] : prof_pending) {
      HMI_CUDA(cudaEventSynchronize(e.second));
      float ms = 0;
      HMI_CUDA(cudaEventElapsedTime(&ms, e.first, e.second));
      prof_ms[cls] += ms;
      prof_cnt[cls] += 1;
      prof_free.push_back(e.first);
      prof_free.push_back(e.second);
    }
    prof_pending.clear();
  }

  uint8_t* store_alloc() {
    if (!free_blocks.empty()) {
      uint8_t* p = free_blocks.back();
      free_blocks.pop_back();
      return p;
    }
    const size_t need = static_cast<size_t>(L) * slot_bytes;
    if (chunk_left < need) {
      const size_t chunk = std::max<size_t>(need, size_t(256) << 20);
      uint8_t* p = host_alloc_local(chunk, numa_node);
      pinned_chunks.push_back({p, chunk});
      chunk_cur = p;
      chunk_left = chunk;
    }
    uint8_t* p = chunk_cur;
    chunk_cur += need;
    chunk_left -= need;
    return p;
  }

  void reap(bool all);
  void build_plans();
  void upload_plot_hash();
  void convert_adapter(const float* src, uint8_t* dst) const;
  // re-associate the down projections of converted host blocks onto ctx (adapter.cu); in place
  void fold_adapters(uint8_t* const* blocks, size_t n);
  int submit(uint32_t n_req, const uint32_t* inst, const uint32_t* tokens_host,
             const uint32_t* tokens_dev, uint32_t stride, const uint32_t* lens_host,
             const uint32_t* lens_dev, uint32_t max_len, float* d_scores_out,
             int32_t* d_labels_out, std::vector<PoolRecord>* records,
             std::vector<int32_t>* record_layer, uint32_t n_new = 0);
  void decode_steps(uint32_t n_req, uint32_t n_new, int S, const LmHead& lm, int wide_head);
  void launch_lm_head(uint32_t n_req, int S, const LmHead& lm, int wide_head, bool gen,
                      float* scores, int32_t* labels);
};

Ctx::~Ctx() {
  if (compute) cudaStreamSynchronize(compute);
  if (copy) cudaStreamSynchronize(copy);
  for (auto& l : layers) {
    if (l.mem) cudaFree(l.mem);
    if (l.mem_fold) cudaFree(l.mem_fold);
  }
  d_stats1.free();
  d_stats2.free();
  qkv_dec.free(); kv_tail.free(); hdec16.free(); hdec32.free(); lm_logits.free();
  gen_tokens.free(); gen_pos.free(); gen_out.free(); gen_logit.free();
  for (auto& [id, h] : lm_heads) {
    if (h.w16) cudaFree(h.w16);
    if (h.bias) cudaFree(h.bias);
    if (h.wT) cudaFree(h.wT);
  }
  for (auto& s : stg) {
    for (void* p : {static_cast<void*>(s.inst), static_cast<void*>(s.tokens),
                    static_cast<void*>(s.lens), static_cast<void*>(s.delta),
                    static_cast<void*>(s.scores), static_cast<void*>(s.labels),
                    static_cast<void*>(s.tags), static_cast<void*>(s.err)})
      if (p) cudaFreeHost(p);
    if (s.done) cudaEventDestroy(s.done);
  }
  for (auto& [p, n] : pinned_chunks) host_free_local(p, n);
  for (auto& [k, p] : ipc_open) cudaIpcCloseMemHandle(p);
  for (auto& [k, g] : dec_graphs) cudaGraphExecDestroy(g);
  for (auto e : ev_layer) cudaEventDestroy(e);
  if (copy2) cudaStreamDestroy(copy2);
  if (ev_fork) cudaEventDestroy(ev_fork);
  if (ev_join) cudaEventDestroy(ev_join);
  d_ready.free();
  for (auto& [c, e] : prof_pending) {
    cudaEventDestroy(e.first);
    cudaEventDestroy(e.second);
  }
  for (auto e : prof_free) cudaEventDestroy(e);
  h16.free(); qkv16.free(); ctx16.free(); a16.free(); mid16.free(); x16.free(); ffn16.free();
  y32.free(); h32.free(); h64.free();
  d_inst.free(); d_tokens.free(); d_lens.free(); d_delta.free(); d_req_version.free();
  d_req_task.free(); d_req_head.free(); d_tile_slot.free(); d_err.free(); d_gather.free();
  d_levels.free(); d_scores.free(); d_labels.free(); d_tags.free();
  d_inst_version.free(); d_inst_task.free(); d_inst_head.free(); d_slot_of.free();
  d_slots.free(); d_parent.free(); d_reps.free(); d_head_arena.free(); d_head_off.free();
  d_head_labels.free(); d_head_kind.free(); arena.free();
  wo32.free(); bo32.free(); fold_in.free(); fold_out.free();
  if (fold_stream) cudaStreamDestroy(fold_stream);
  if (compute) cudaStreamDestroy(compute);
  if (copy) cudaStreamDestroy(copy);
}

// Device layout of one (task, layer) adapter slot:
//   [Wd^T: r_pad x d 16-bit][Wu^T: d x r_pad 16-bit][bd: r_pad f32][bu: d f32]
// rows beyond r are zero, so the padded GEMMs add exact zeros.
void Ctx::convert_adapter(const float* src, uint8_t* dst) const {
  const int prec = static_cast<int>(opt.precision);
  for (int l = 0; l < L; ++l) {
    const float* wd = src;
    const float* bd = wd + static_cast<size_t>(d) * r;
    const float* wu = bd + r;
    const float* bu = wu + static_cast<size_t>(r) * d;
    src = bu + d;
    uint8_t* slot = dst + static_cast<size_t>(l) * slot_bytes;
    uint16_t* wdt = reinterpret_cast<uint16_t*>(slot);
    uint16_t* wut = wdt + static_cast<size_t>(r_pad) * d;
    float* bdd = reinterpret_cast<float*>(wut + static_cast<size_t>(d) * r_pad);
    float* bud = bdd + r_pad;
    std::memset(slot, 0, slot_bytes);
    // transposes in 32 x 32 tiles (both sides stay in L1)
    constexpr int kT = 32;
    for (int j0 = 0; j0 < r; j0 += kT)
      for (int i0 = 0; i0 < d; i0 += kT)
        for (int j = j0; j < std::min(j0 + kT, r); ++j)
          for (int i = i0; i < std::min(i0 + kT, d); ++i)
            wdt[static_cast<size_t>(j) * d + i] = f2h(wd[static_cast<size_t>(i) * r + j], prec);
    for (int i0 = 0; i0 < d; i0 += kT)
      for (int j0 = 0; j0 < r; j0 += kT)
        for (int i = i0; i < std::min(i0 + kT, d); ++i)
          for (int j = j0; j < std::min(j0 + kT, r); ++j)
            wut[static_cast<size_t>(i) * r_pad + j] = f2h(wu[static_cast<size_t>(j) * d + i], prec);
    for (int j = 0; j < r; ++j) bdd[j] = bd[j];
    for (int i = 0; i < d; ++i) bud[i] = bu[i];
  }
}

void Ctx::fold_adapters(uint8_t* const* blocks, size_t n) {
  if (n == 0) return;
  HMI_CUDA(cudaSetDevice(device));
  const size_t per = static_cast<size_t>(L) * slot_bytes;
  if (fold_cap == 0) {
    fold_cap = std::max<size_t>(1, (64ull << 20) / per);
    fold_in.alloc(fold_cap * per);
    fold_out.alloc(fold_cap * per);
    HMI_CUDA(cudaStreamCreateWithFlags(&fold_stream, cudaStreamNonBlocking));
  }
  const size_t off_bd = static_cast<size_t>(r_pad) * d * 2 * 2;
  for (size_t b0 = 0; b0 < n; b0 += fold_cap) {
    const size_t nb = std::min(fold_cap, n - b0);
    for (size_t k = 0; k < nb; ++k)
      HMI_CUDA(cudaMemcpyAsync(fold_in.p + k * per, blocks[b0 + k], per, cudaMemcpyHostToDevice,
                               fold_stream));
    launch_adapter_fold(fold_in.p, fold_out.p, static_cast<int>(nb * L), wo32.p, bo32.p, L, d,
                        r_pad, slot_bytes, off_bd, static_cast<int>(opt.precision), fold_stream);
    for (size_t k = 0; k < nb; ++k) {  // Wc^T and bc of every layer back into the host block
      HMI_CUDA(cudaMemcpy2DAsync(blocks[b0 + k], slot_bytes, fold_out.p + k * per, slot_bytes,
                                 static_cast<size_t>(r_pad) * d * 2, L, cudaMemcpyDeviceToHost,
                                 fold_stream));
      HMI_CUDA(cudaMemcpy2DAsync(blocks[b0 + k] + off_bd, slot_bytes, fold_out.p + k * per + off_bd,
                                 slot_bytes, static_cast<size_t>(r_pad) * 4, L,
                                 cudaMemcpyDeviceToHost, fold_stream));
    }
    HMI_CUDA(cudaStreamSynchronize(fold_stream));
  }
}

void Ctx::build_plans() {
  attn.clear();
  for (int l = 0; l < (kv ? L : 1); ++l)
    attn.push_back(make_attention_plan(qkv_at(l), ctx16.p, max_rows, d, static_cast<int>(opt.precision)));
  const int sms = device_sm_count();
  {  // GEMM statistics producers emit one partial per 64-column group of the row; the fused
     // adapter one per column half
    const int mt = max_rows / 128;
    stats1_bn = pick_bn(d, mt, sms);
    stats2_bn = pick_bn(d, mt, sms, true);
    stats1_n = d / 64;
    stats2_n = d / 64;
    HMI_CHECK(d % 64 == 0 && d / 64 <= kStatsLd, HMI_CONFIG_ERROR,
              "hidden size too wide for the LayerNorm statistics buffer");
  }
  const int m_tiles = max_rows / 128;
  const int prec = static_cast<int>(opt.precision);
  const size_t off_wu = static_cast<size_t>(r_pad) * d * 2;
  const size_t off_bd = off_wu + static_cast<size_t>(d) * r_pad * 2;
  const size_t off_bu = off_bd + static_cast<size_t>(r_pad) * 4;
  const uint32_t n_slots = pool->physical_slots();
  for (int l = 0; l < L; ++l) {
    LayerDev& w = layers[l];
    GemmSpec s;
    s.precision = prec;
    s.a_rows = max_rows;
    // QKV
    s.a = h16.p; s.a_ld = d; s.K = d;
    s.b = w.wqkv; s.N = 3 * d; s.groups = 1; s.b_ld = d; s.b_group_stride_bytes = size_t(3) * d * d * 2;
    s.bias = w.bqkv; s.bias_group_stride = 0; s.tile_slot = nullptr;
    s.res0 = s.res1 = nullptr; s.res_ld = 0;
    s.c = qkv_at(l); s.c_ld = 3 * d; s.epi = 0; s.cta2 = true;
    s.bn = pick_bn(3 * d, m_tiles, sms, true);
    w.qkv = make_gemm_plan(s);
    // O projection
    s.a = ctx16.p; s.a_ld = d; s.K = d;
    s.b = w.wo; s.N = d; s.b_ld = d; s.b_group_stride_bytes = size_t(d) * d * 2;
    s.bias = w.bo; s.c = a16.p; s.c_ld = d; s.epi = 0; s.bn = pick_bn(d, m_tiles, sms, true);
    w.oproj = make_gemm_plan(s);
    // adapter down (grouped, folded weights): mid = relu(ctx . Wc + bc) = relu(a . Wd + bd)
    s.a = ctx16.p; s.a_ld = d; s.K = d;
    s.b = arena.p; s.N = r_pad; s.groups = static_cast<int>(n_slots); s.b_ld = d;
    s.b_group_stride_bytes = slot_bytes;
    s.bias = reinterpret_cast<const float*>(arena.p + off_bd);
    s.bias_group_stride = static_cast<long long>(slot_bytes / 4);
    s.tile_slot = d_tile_slot.p + static_cast<size_t>(l) * tile_stride;
    s.c = mid16.p; s.c_ld = r_pad; s.epi = kEpiRelu; s.bn = r_pad;
    w.ad_down = make_gemm_plan(s);
    // adapter up (grouped) + skip (a) + residual (h): y = mid . Wu + bu + a + h
    s.a = mid16.p; s.a_ld = r_pad; s.K = r_pad;
    s.b = arena.p + off_wu; s.N = d; s.b_ld = r_pad;
    s.bias = reinterpret_cast<const float*>(arena.p + off_bu);
    s.res0 = a16.p; s.res1 = h16.p; s.res_ld = d;
    s.c = y32.p; s.c_ld = d; s.epi = kEpiRes2 | kEpiOutF32; s.cta2 = false;
    s.bn = pick_bn(d, m_tiles, sms);
    w.ad_up = make_gemm_plan(s);
    // FFN1: relu(x . W1 + b1)
    s.a = x16.p; s.a_ld = d; s.K = d;
    s.b = w.w1; s.N = f; s.groups = 1; s.b_ld = d; s.b_group_stride_bytes = size_t(f) * d * 2;
    s.bias = w.b1; s.bias_group_stride = 0; s.tile_slot = nullptr;
    s.res0 = s.res1 = nullptr;
    s.c = ffn16.p; s.c_ld = f; s.epi = kEpiRelu; s.cta2 = true;
    s.bn = pick_bn(f, m_tiles, sms, true);
    w.ffn1 = make_gemm_plan(s);
    // FFN2 + residual: y = ffn . W2 + b2 + x
    s.a = ffn16.p; s.a_ld = f; s.K = f;
    s.b = w.w2; s.N = d; s.b_ld = f; s.b_group_stride_bytes = size_t(d) * f * 2;
    s.bias = w.b2; s.res0 = x16.p; s.res_ld = d;
    s.c = y32.p; s.c_ld = d; s.epi = kEpiRes1 | kEpiOutF32; s.bn = pick_bn(d, m_tiles, sms, true);
    w.ffn2 = make_gemm_plan(s);
    {
      // LayerNorm folding. Buffers hold PRE-norm rows: x16 = y1 (pre-LN1), h16 = y2 (pre-LN2
      // of layer l-1; h0 for l = 0); d_stats1/2 their partial row sums.
      const LayerDev* prev = l > 0 ? &layers[l - 1] : nullptr;
      const float inv_d = 1.0f / static_cast<float>(d);
      if (prev) {  // QKV on LN2_{l-1}(y2): gamma folded into W, mean corrected in the epilogue
        GemmSpec q;
        q.precision = prec;
        q.a_rows = max_rows;
        q.a = h16.p; q.a_ld = d; q.K = d;
        q.b = w.wqkv_f; q.N = 3 * d; q.groups = 1; q.b_ld = d;
        q.b_group_stride_bytes = size_t(3) * d * d * 2;
        q.bias = w.bqkv_f; q.c = qkv_at(l); q.c_ld = 3 * d; q.epi = kEpiFoldLN; q.cta2 = true;
        q.a_stats = d_stats2.p; q.a_stats_n = stats2_n; q.colsum = w.cs_qkv; q.inv_n = inv_d;
        q.bn = pick_bn(3 * d, m_tiles, sms, true);
        w.qkv = make_gemm_plan(q);
      }
      {  // adapter up: y1 = mid.Wu + bu + a + LN2_{l-1}(y2)  (+ partial stats of y1)
        GemmSpec u;
        u.precision = prec;
        u.a_rows = max_rows;
        u.a = mid16.p; u.a_ld = r_pad; u.K = r_pad;
        u.b = arena.p + off_wu; u.N = d; u.groups = static_cast<int>(n_slots); u.b_ld = r_pad;
        u.b_group_stride_bytes = slot_bytes;
        u.bias = reinterpret_cast<const float*>(arena.p + off_bu);
        u.bias_group_stride = static_cast<long long>(slot_bytes / 4);
        u.tile_slot = d_tile_slot.p + static_cast<size_t>(l) * tile_stride;
        u.res0 = a16.p; u.res1 = h16.p; u.res_ld = d;
        u.c = x16.p; u.c_ld = d;
        u.epi = kEpiRes2 | kEpiStats | (prev ? kEpiRes1LN : 0) | (stats1_bn <= 192 ? kEpiResTma : 0);
        u.stats_out = d_stats1.p; u.stats_ld = kStatsLd;
        if (prev) {
          u.r_stats = d_stats2.p; u.r_stats_n = stats2_n;
          u.r_gamma = prev->ln2g; u.r_beta = prev->ln2b; u.inv_n = inv_d;
        }
        u.bn = stats1_bn;
        w.ad_up = make_gemm_plan(u);
        if (oproj_ext) {
          // y1 = [ctx | mid] . [Wo ; Wu_tenant] + bo + bu + LN2_{l-1}(y2)  (+ partial stats of y1)
          GemmSpec o;
          o.precision = prec;
          o.a_rows = max_rows;
          o.a = ctx16.p; o.a_ld = d; o.K = d;
          o.b = w.wo; o.N = d; o.groups = 1; o.b_ld = d; o.b_group_stride_bytes = size_t(d) * d * 2;
          o.bias = w.bo; o.tile_slot = u.tile_slot;
          o.res0 = h16.p; o.res_ld = d; o.c = x16.p; o.c_ld = d;
          o.epi = kEpiExt | kEpiRes1 | kEpiStats | (prev ? kEpiRes0LN : 0); o.cta2 = true;
          o.stats_out = d_stats1.p; o.stats_ld = kStatsLd;
          if (prev) {
            o.r_stats = d_stats2.p; o.r_stats_n = stats2_n;
            o.r_gamma = prev->ln2g; o.r_beta = prev->ln2b; o.inv_n = inv_d;
          }
          o.ext_a = mid16.p; o.ext_k = r_pad;
          o.ext_b = arena.p + off_wu; o.ext_b_ld = r_pad; o.ext_groups = static_cast<int>(n_slots);
          o.ext_b_stride = slot_bytes;
          o.ext_bias = reinterpret_cast<const float*>(arena.p + off_bu);
          o.ext_bias_stride = static_cast<long long>(slot_bytes / 4);
          o.bn = pick_bn(d, m_tiles, sms, true);
          w.oproj = make_gemm_plan(o);
        }
      }
      {  // FFN1 on LN1(y1)
        GemmSpec g;
        g.precision = prec;
        g.a_rows = max_rows;
        g.a = x16.p; g.a_ld = d; g.K = d;
        g.b = w.w1_f; g.N = f; g.groups = 1; g.b_ld = d; g.b_group_stride_bytes = size_t(f) * d * 2;
        g.bias = w.b1_f; g.c = ffn16.p; g.c_ld = f; g.epi = kEpiRelu | kEpiFoldLN; g.cta2 = true;
        g.a_stats = d_stats1.p; g.a_stats_n = stats1_n; g.colsum = w.cs_1; g.inv_n = inv_d;
        g.bn = pick_bn(f, m_tiles, sms, true);
        w.ffn1 = make_gemm_plan(g);
      }
      {  // FFN2: y2 = ffn.W2 + b2 + LN1(y1)  (+ partial stats of y2)
        GemmSpec g;
        g.precision = prec;
        g.a_rows = max_rows;
        g.a = ffn16.p; g.a_ld = f; g.K = f;
        g.b = w.w2; g.N = d; g.groups = 1; g.b_ld = f; g.b_group_stride_bytes = size_t(d) * f * 2;
        g.bias = w.b2; g.res0 = x16.p; g.res_ld = d; g.c = h16.p; g.c_ld = d;
        g.epi = kEpiRes1 | kEpiRes0LN | kEpiStats; g.cta2 = true;
        g.stats_out = d_stats2.p; g.stats_ld = kStatsLd;
        g.r_stats = d_stats1.p; g.r_stats_n = stats1_n; g.r_gamma = w.ln1g; g.r_beta = w.ln1b;
        g.inv_n = inv_d;
        g.bn = stats2_bn;
        w.ffn2 = make_gemm_plan(g);
      }
    }
  }
  // single-row decode steps: unfolded weights, explicit LayerNorms, 1-CTA tiles
  dec.clear();
  if (kv) {
    const int mt = Bp / 128;
    auto dec_plan = [&](const GemmSpec& g) {
      try {
        return make_dec_gemm_plan(g, mt);
      } catch (const HmiError& e) {
        if (e.code != HMI_CONFIG_ERROR) throw;
        return DecGemmPlan{};  // no (tile, K split) fits: the K1 plan serves this GEMM
      }
    };
    for (int l = 0; l < L; ++l) {
      LayerDev& w = layers[l];
      DecPlans dp;
      GemmSpec s;
      s.precision = prec;
      s.a_rows = Bp;
      s.a = h16.p; s.a_ld = d; s.K = d;
      s.b = w.wqkv; s.N = 3 * d; s.b_ld = d; s.b_group_stride_bytes = size_t(3) * d * d * 2;
      s.bias = w.bqkv; s.c = qkv_dec.p; s.c_ld = 3 * d; s.epi = 0;
      s.bn = pick_bn(3 * d, mt, sms);
      dp.qkv = make_gemm_plan(s);
      dp.kqkv = dec_plan(s);
      s.a = ctx16.p; s.b = w.wo; s.N = d; s.b_group_stride_bytes = size_t(d) * d * 2;
      s.bias = w.bo; s.c = a16.p; s.c_ld = d; s.bn = pick_bn(d, mt, sms);
      dp.oproj = make_gemm_plan(s);
      dp.koproj = dec_plan(s);
      s.a = x16.p; s.b = w.w1; s.N = f; s.b_group_stride_bytes = size_t(f) * d * 2;
      s.bias = w.b1; s.c = ffn16.p; s.c_ld = f; s.epi = kEpiRelu; s.bn = pick_bn(f, mt, sms);
      dp.ffn1 = make_gemm_plan(s);
      dp.kffn1 = dec_plan(s);
      s.a = ffn16.p; s.a_ld = f; s.K = f; s.b = w.w2; s.N = d; s.b_ld = f;
      s.b_group_stride_bytes = size_t(d) * f * 2; s.bias = w.b2; s.res0 = x16.p; s.res_ld = d;
      s.c = y32.p; s.c_ld = d; s.epi = kEpiRes1 | kEpiOutF32; s.bn = pick_bn(d, mt, sms);
      dp.ffn2 = make_gemm_plan(s);
      dp.kffn2 = dec_plan(s);
      dp.attn = make_attn_decode_maps(qkv_at(l), max_rows,
                                      kv_tail.p + static_cast<size_t>(l) * opt.max_batch *
                                                      opt.max_new_tokens * 2 * d,
                                      static_cast<int>(opt.max_batch),
                                      static_cast<int>(opt.max_new_tokens), d, prec);
      dec.push_back(dp);
    }
  }
}

void Ctx::build_lm_plan(LmHead& h) {
  GemmSpec s;
  s.precision = static_cast<int>(opt.precision);
  s.a_rows = Bp;
  s.a = hdec16.p; s.a_ld = d; s.K = d;
  s.b = h.w16; s.N = h.V_pad; s.b_ld = d; s.b_group_stride_bytes = static_cast<size_t>(h.V_pad) * d * 2;
  s.bias = h.bias; s.c = lm_logits.p; s.c_ld = static_cast<int>(lm_logits.n / Bp);
  s.epi = kEpiOutF32;
  // the pair kernel: both 128-row halves of a 256-row batch share each streamed weight tile
  // (the 1-CTA form read the 77 MB GPT-2 head once per 128-row tile, at BN = 64 re-reading
  // the rows 786 times)
  s.cta2 = true;
  s.bn = pick_bn(h.V_pad, Bp / 128, device_sm_count(), true);
  h.plan = make_gemm_plan(s);
}

void Ctx::upload_plot_hash() {
  HMI_CUDA(cudaStreamSynchronize(compute));
  if (d_slots.n != h_slots.size()) d_slots.alloc(h_slots.size());
  HMI_CUDA(cudaMemcpy(d_slots.p, h_slots.data(), h_slots.size() * sizeof(PlotSlot),
                      cudaMemcpyHostToDevice));
  HMI_CUDA(cudaMemcpy(d_parent.p, h_parent.data(), h_parent.size() * sizeof(int32_t),
                      cudaMemcpyHostToDevice));
}

void Ctx::reap(bool all) {
  while (!inflight.empty()) {
    Inflight& f = inflight.front();
    if (all) {
      HMI_CUDA(cudaEventSynchronize(f.done));
    } else if (cudaEventQuery(f.done) != cudaSuccess) {
      break;
    }
    pool->unpin(f.tasks);
    Staging& st = stg[f.staging];
    // a finished batch nobody waits on (infer_batch_device): latch its device-side error
    // for hmi_gpu_synchronize / the next asynchronous submit; synchronous callers have read
    // and cleared theirs already
    if (!st.held) {
      if (*st.err != 0 && sticky_err == 0) sticky_err = *st.err;
      *st.err = 0;
    }
    st.busy = false;
    inflight.pop_front();
  }
}

int Ctx::submit(uint32_t n_req, const uint32_t* inst, const uint32_t* tokens_host,
                const uint32_t* tokens_dev, uint32_t stride, const uint32_t* lens_host,
                const uint32_t* lens_dev, uint32_t max_len, float* d_scores_out,
                int32_t* d_labels_out, std::vector<PoolRecord>* records,
                std::vector<int32_t>* record_layer, uint32_t n_new) {
  HMI_CHECK(n_req >= 1 && n_req <= opt.max_batch, HMI_DIMENSION_ERROR,
            "batch size must be in [1, max_batch]");
  const double trace_host_a = trace_on ? host_ms() : 0.0;
  HMI_CHECK(!stg[stg_next].held, HMI_CAPACITY_ERROR,
            "too many outstanding submitted batches: wait on the oldest ticket first");
  const bool gen = n_new > 0;
  HMI_CHECK(!gen || (kv && n_new <= opt.max_new_tokens), HMI_CONFIG_ERROR,
            "generation needs max_new_tokens >= n_new (causal model)");
  const bool sync_mode = opt.pipeline_mode == 0;
  const bool fine = opt.pipeline_mode == 2;
  reap(sync_mode);

  // ---- host routing mirror (InstanceTable) and request validation
  std::vector<uint32_t> tasks(n_req);
  for (uint32_t i = 0; i < n_req; ++i) {
    const uint32_t k = inst[i];
    if (k >= h_inst_task.size() || h_inst_task[k] < 0) {
      throw HmiError(HMI_ROUTING_ERROR, "instance " + std::to_string(k) + " is not bound");
    }
    tasks[i] = static_cast<uint32_t>(h_inst_task[k]);
  }
  // wide lm heads of this batch (at most one; generation needs every request on it)
  int wide_head = -1;
  for (uint32_t i = 0; i < n_req; ++i) {
    const int hd = h_inst_head[inst[i]];
    const bool wide = lm_heads.count(hd) != 0;
    if (wide) {
      HMI_CHECK(wide_head < 0 || wide_head == hd, HMI_CONFIG_ERROR,
                "a batch may use at most one wide lm head");
      wide_head = hd;
    }
    HMI_CHECK(!gen || wide, HMI_CONFIG_ERROR, "generation needs every request bound to a wide lm head");
  }
  HMI_CHECK(!gen || lm_heads.at(wide_head).V <= static_cast<int>(cfg.vocab_size), HMI_CONFIG_ERROR,
            "generation: the lm head emits ids outside the vocabulary");
  if (lens_host) {
    max_len = 0;
    for (uint32_t i = 0; i < n_req; ++i) {
      HMI_CHECK(lens_host[i] >= 1 && lens_host[i] <= stride, HMI_DIMENSION_ERROR,
                "request length must be in [1, stride]");
      max_len = std::max(max_len, lens_host[i]);
      for (uint32_t p = 0; p < lens_host[i]; ++p) {
        if (tokens_host[static_cast<size_t>(i) * stride + p] >= cfg.vocab_size) {
          throw HmiError(HMI_VOCABULARY_ERROR, "token id outside vocabulary");
        }
      }
    }
  }
  HMI_CHECK(max_len >= 1 && max_len <= static_cast<uint32_t>(S_max), HMI_DIMENSION_ERROR,
            "request length exceeds max_seq");
  const int S = static_cast<int>((max_len + 127) / 128 * 128);
  const int rows = static_cast<int>(n_req) * S;
  const int tiles_per_req = S / 128;

  // ---- residency decisions (stage_prefetch)
  std::vector<uint32_t> uniq;
  {
    std::set<uint32_t> seen;
    for (uint32_t t : tasks)
      if (seen.insert(t).second) uniq.push_back(t);
  }
  std::vector<std::vector<std::pair<uint32_t, int32_t>>> loads(L);  // per layer (task, slot)
  std::vector<int32_t> delta;
  auto absorb = [&](std::vector<PoolRecord>& recs, int layer_tag) {
    for (auto& rec : recs) {
      for (const PoolFree& fr : rec.freed) {
        delta.push_back(static_cast<int32_t>(fr.task * L + fr.layer));
        delta.push_back(-1);
      }
      for (const PoolLoad& ld : rec.loads) {
        loads[ld.layer].push_back({rec.task, ld.slot});
        delta.push_back(static_cast<int32_t>(rec.task * L + ld.layer));
        delta.push_back(ld.slot);
      }
      if (records) {
        records->push_back(rec);
        record_layer->push_back(layer_tag);
      }
    }
  };
  // Every decision the pool makes for this batch is absorbed, including those of an attempt
  // that failed on pinned blockers (take_partial): the retry sees those tasks as hits, so
  // their copies and slot-table deltas must come from here. If submit throws before the
  // batch is enqueued, the guard rolls the placements back (their copies were never issued)
  // and releases the pins.
  struct Undo {
    SlotPool* pool;
    std::vector<std::pair<uint32_t, uint32_t>> placed;  // (task, layer)
    const std::vector<uint32_t>* pinned = nullptr;
    bool armed = true;
    ~Undo() {
      if (!armed) return;
      if (pinned) pool->unpin(*pinned);
      for (auto it = placed.rbegin(); it != placed.rend(); ++it) pool->unload(it->first, it->second);
    }
  } undo{pool.get(), {}};
  auto absorb_all = [&](std::vector<PoolRecord>&& recs, int layer_tag) {
    for (const auto& rec : recs)
      for (const PoolLoad& ld : rec.loads) undo.placed.push_back({rec.task, ld.layer});
    absorb(recs, layer_tag);
  };
  if (!fine) {
    for (;;) {
      try {
        absorb_all(pool->ensure_resident(uniq), -1);
        break;
      } catch (const HmiError& e) {
        absorb_all(pool->take_partial(), -1);
        // a pinned in-flight working set blocks the load: retire the oldest batch and retry
        if (e.code != HMI_CAPACITY_ERROR || inflight.empty()) throw;
        HMI_CUDA(cudaEventSynchronize(inflight.front().done));
        reap(false);
      }
    }
  } else {
    for (int l = 0; l < L; ++l) {
      for (;;) {
        std::optional<std::vector<PoolRecord>> recs;
        try {
          recs = pool->try_ensure_layer_resident(uniq, static_cast<uint32_t>(l));
        } catch (...) {
          absorb_all(pool->take_partial(), l);
          throw;
        }
        absorb_all(pool->take_partial(), l);
        if (recs) {
          absorb_all(std::move(*recs), l);
          break;
        }
        if (inflight.empty()) {
          throw HmiError(HMI_CAPACITY_ERROR, "pinned working set blocks adapter load");
        }
        HMI_CUDA(cudaEventSynchronize(inflight.front().done));
        reap(false);
      }
    }
  }
  pool->pin(uniq);
  undo.pinned = &uniq;

  // ---- staging buffer for this batch
  const int si = stg_next;
  stg_next = (stg_next + 1) % kStaging;
  Staging& st = stg[si];
  if (st.busy) {
    while (stg[si].busy) {
      HMI_CUDA(cudaEventSynchronize(inflight.front().done));
      reap(false);
    }
  }
  HMI_CHECK(delta.size() / 2 <= d_delta.n / 2, HMI_SCHEDULING_BUG, "slot delta overflow");
  std::memcpy(st.inst, inst, n_req * sizeof(uint32_t));
  if (!delta.empty()) std::memcpy(st.delta, delta.data(), delta.size() * sizeof(int32_t));
  if (tokens_host) {
    for (uint32_t i = 0; i < n_req; ++i) {
      std::memcpy(st.tokens + static_cast<size_t>(i) * S, tokens_host + static_cast<size_t>(i) * stride,
                  std::min<uint32_t>(stride, S) * sizeof(uint32_t));
      st.lens[i] = static_cast<int32_t>(lens_host[i]);
    }
  }

  // fine mode: device-side readiness flags (see d_ready), waited on by the first reader of
  // the layer's slots (the tenant-grouped down GEMM)
  const bool device_ready = fine && write_value32 != nullptr;
  const uint32_t seq = ++ready_seq;
  // ---- copy stream: adapter H2D into HBM slots, one event per layer
  // Whole-task misses are one contiguous copy: the pool places a task's layers in consecutive
  // slots of a block (slot_pool.hpp) and the host store keeps them consecutive, so each run of
  // consecutive layers in consecutive slots of one task is one cudaMemcpyAsync (per-transfer
  // setup, not PCIe, bounds slot-sized copies: ~27 GB/s at 200 KB, ~47 at 1.2 MB). Every
  // layer's event (and device flag) follows all of the batch's copies.
  copy_items.clear();
  for (int l = 0; l < L; ++l)
    for (const auto& ld : loads[l]) copy_items.push_back({ld.first, static_cast<uint32_t>(l), ld.second});
  std::sort(copy_items.begin(), copy_items.end(), [](const CopyItem& a, const CopyItem& b) {
    return a.task != b.task ? a.task < b.task : a.layer < b.layer;
  });
  for (int l = 0; l < L; ++l) traced(kStagePrefetch, l, kWorkerIo, copy, [&] {
    if (l == 0) {
      auto src = [&](const CopyItem& it) { return store[it.task] + static_cast<size_t>(it.layer) * slot_bytes; };
      const bool two = copy_items.size() > static_cast<size_t>(L);
      if (two) {
        HMI_CUDA(cudaEventRecord(ev_fork, copy));
        HMI_CUDA(cudaStreamWaitEvent(copy2, ev_fork, 0));
      }
      int run = 0;
      for (size_t i = 0; i < copy_items.size(); ++run) {
        // a run: consecutive slot images at consecutive host and device addresses (a task's
        // layers in its block; consecutively registered tasks in consecutive blocks too)
        size_t j = i + 1;
        while (j < copy_items.size() && src(copy_items[j]) == src(copy_items[j - 1]) + slot_bytes &&
               copy_items[j].slot == copy_items[j - 1].slot + 1)
          ++j;
        HMI_CUDA(cudaMemcpyAsync(arena.p + static_cast<size_t>(copy_items[i].slot) * slot_bytes,
                                 src(copy_items[i]), (j - i) * slot_bytes, cudaMemcpyHostToDevice,
                                 two && (run & 1) ? copy2 : copy));
        ++n_copies;  // host -> HBM transfers
        i = j;
      }
      if (two) {
        HMI_CUDA(cudaEventRecord(ev_join, copy2));
        HMI_CUDA(cudaStreamWaitEvent(copy, ev_join, 0));
      }
      bytes_copied += copy_items.size() * slot_bytes;
    }
    HMI_CUDA(cudaEventRecord(ev_layer[l], copy));
    if (device_ready) {
      const CUresult r = write_value32(reinterpret_cast<CUstream>(copy),
                                       reinterpret_cast<CUdeviceptr>(d_ready.p + l), seq, 0);
      HMI_CHECK(r == CUDA_SUCCESS, HMI_CUDA_ERROR, "cuStreamWriteValue32 failed");
    }
  });

  // ---- compute stream
  cudaStream_t s = compute;
  if (sync_mode || !fine) {
    // sync / coarse: every layer's adapters resident before this batch computes
    HMI_CUDA(cudaStreamWaitEvent(s, ev_layer[L - 1], 0));
  }
  timed(P_H2D, s, [&] {
    // inputs fetched by a kernel (SM loads over PCIe from the pinned staging): copy-engine
    // transfers on this stream would queue behind later batches' adapter copies
    FetchArgs fa;
    fa.inst = st.inst; fa.d_inst = d_inst.p; fa.n_inst = static_cast<int>(n_req);
    fa.d_tokens = d_tokens.p; fa.n_req = static_cast<int>(n_req); fa.S = S;
    if (tokens_host) {
      fa.tokens = st.tokens; fa.src_stride = S;
      fa.lens = st.lens;
    } else {
      fa.tokens = tokens_dev; fa.src_stride = static_cast<int>(stride);
      fa.lens = reinterpret_cast<const int32_t*>(lens_dev);
    }
    fa.d_lens = d_lens.p;
    fa.delta = st.delta; fa.d_delta = d_delta.p; fa.n_delta = static_cast<int>(delta.size());
    fa.d_err = d_err.p;
    launch_fetch_inputs(fa, s);
  });
  timed(P_ROUTE, s, [&] {
    if (!delta.empty()) launch_apply_deltas(d_slot_of.p, d_delta.p, static_cast<int>(delta.size() / 2), s);
    launch_route(d_inst.p, static_cast<int>(n_req), d_inst_version.p, d_inst_task.p, d_inst_head.p,
                 static_cast<int>(h_inst_task.size()), d_slot_of.p, L, tiles_per_req, tile_stride,
                 d_req_version.p,
                 d_req_task.p, d_req_head.p, d_tile_slot.p, d_err.p, s);
  });
  PlotDev P;
  P.slots = d_slots.p;
  P.mask = h_slots.empty() ? 0 : h_slots.size() - 1;
  P.parent = d_parent.p;
  P.max_versions = static_cast<int>(h_parent.size());
  P.reps = d_reps.p;
  P.ngram = ngram;
  P.d = d;
  P.max_depth = 1;
  for (size_t v = 0; v < h_parent.size(); ++v) {
    if (h_parent[v] == -2) continue;
    int depth = 1;
    for (int32_t u = h_parent[v]; u >= 0; u = h_parent[u]) ++depth;
    P.max_depth = std::max(P.max_depth, depth);
  }
  const int causal = cfg.mode == 1 ? 1 : 0;
  const int prec = static_cast<int>(opt.precision);
  traced(kStageRetrieve, -1, kWorkerCompute, s, [&] {
    timed(P_RETRIEVE, s, [&] {
      launch_retrieve(P, d_tokens.p, d_lens.p, d_req_version.p, static_cast<int>(n_req), S, causal,
                      h16.p, prec, (debug_flags & 1) ? h64.p : nullptr, d_gather.p, d_levels.p,
                      d_err.p, s);
    });
  });
  for (int l = 0; l < L; ++l) traced(kStageCompute, l, kWorkerCompute, s, [&] {
    LayerDev& w = layers[l];
    timed(P_QKV, s, [&] { launch_gemm(w.qkv, rows, s); });
    timed(P_ATTN, s, [&] {
      const AttnPlan& ap = attn[kv ? l : 0];
      if (S == 128) {
        launch_attention_tc(ap, d_lens.p, static_cast<int>(n_req), heads, causal, s);
      } else if (attention_long_tc_ok(S)) {
        launch_attention_long_tc(ap, d_lens.p, static_cast<int>(n_req), S, heads, causal, s);
      } else {  // padded lengths beyond 512 (TMEM holds the scores of 4 key blocks of 128)
        launch_attention(qkv_at(l), ctx16.p, d_lens.p, static_cast<int>(n_req), S, d, heads, causal,
                         prec, s);
      }
    });
    if (fine && !device_ready) HMI_CUDA(cudaStreamWaitEvent(s, ev_layer[l], 0));
    // mid = ReLU(ctx . Wc + bc): the first reader of this layer's slots
    timed(P_AD_DOWN, s, [&] {
      launch_gemm(w.ad_down, rows, s, device_ready ? d_ready.p + l : nullptr, seq, d_err.p);
    });
    if (oproj_ext) {  // O projection with the tenants' up projections as extra K blocks
      timed(P_OPROJ, s, [&] { launch_gemm(w.oproj, rows, s); });
    } else {  // r > 64 or d not a multiple of 128: O projection, then the grouped up GEMM
      timed(P_OPROJ, s, [&] { launch_gemm(w.oproj, rows, s); });
      timed(P_AD_UP, s, [&] { launch_gemm(w.ad_up, rows, s); });
    }
    timed(P_FFN1, s, [&] { launch_gemm(w.ffn1, rows, s); });
    timed(P_FFN2, s, [&] { launch_gemm(w.ffn2, rows, s); });
  });
  HeadDev H;
  H.arena = d_head_arena.p;
  H.offset = d_head_off.p;
  H.labels = d_head_labels.p;
  H.kind = d_head_kind.p;
  float* scores_dst = d_scores_out ? d_scores_out : d_scores.p;
  int32_t* labels_dst = d_labels_out ? d_labels_out : d_labels.p;
  if (wide_head >= 0 && !gen) {
    HMI_CUDA(cudaMemsetAsync(scores_dst, 0, static_cast<size_t>(n_req) * opt.max_labels * 4, s));
  }
  if (!gen) timed(P_HEAD, s, [&] {
    // the head applies the last layer's LN2 to its pre-norm row
    H.y16 = h16.p;
    H.ln_g = layers[L - 1].ln2g;
    H.ln_b = layers[L - 1].ln2b;
    H.bf16 = prec;
    if (debug_flags & 2) {
      launch_normalize_rows(h16.p, d_stats2.p, stats2_n, 1.0f / d, layers[L - 1].ln2g,
                            layers[L - 1].ln2b, h32.p, rows, d, prec, s);
    }
    launch_head(H, h32.p, d_req_head.p, d_lens.p, static_cast<int>(n_req), S, d,
                static_cast<int>(opt.max_labels), scores_dst, labels_dst, d_tags.p, s);
  });
  if (wide_head >= 0) {
    const LmHead& lm = lm_heads.at(wide_head);
    timed(P_HEAD, s, [&] { launch_lm_head(n_req, S, lm, wide_head, gen, scores_dst, labels_dst); });
    if (gen) decode_steps(n_req, n_new, S, lm, wide_head);
  }
  if (!d_scores_out) {
    timed(P_D2H, s, [&] {
      HMI_CUDA(cudaMemcpyAsync(st.scores, d_scores.p, static_cast<size_t>(n_req) * opt.max_labels * sizeof(float),
                               cudaMemcpyDeviceToHost, s));
      HMI_CUDA(cudaMemcpyAsync(st.labels, d_labels.p, n_req * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    });
  }
  HMI_CUDA(cudaMemcpyAsync(st.err, d_err.p, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  HMI_CUDA(cudaEventRecord(st.done, s));
  if (trace_on) {  // head + D2H (compute), then the host-side submit interval (cpu)
    TraceEv e{n_batches, kStageHead, -1, kWorkerCompute};
    HMI_CUDA(cudaEventCreate(&e.a));
    e.b = nullptr;
    HMI_CUDA(cudaEventRecord(e.a, s));  // marks the end; start = the last layer's end
    trace_evs.push_back(e);
    TraceEv h{n_batches, kStageHost, -1, kWorkerCpu};
    h.host_a = trace_host_a;
    h.host_b = host_ms();
    trace_evs.push_back(h);
  }
  st.busy = true;
  inflight.push_back(Inflight{st.done, si, uniq});
  undo.armed = false;
  last_n = n_req;
  const uint64_t per_layer = oproj_ext ? 6ull : 7ull;
  // fetch_inputs + route + retrieve (+ apply_deltas) + layers + head
  n_launches += (delta.empty() ? 0 : 1) + 3 + (gen ? 0 : 1) + per_layer * L;
  if (wide_head >= 0) n_launches += 3 + (gen ? (n_new - 1ull) * (3 + 7ull * L) : 0);
  ++n_batches;
  last_S = static_cast<uint32_t>(S);
  return si;
}

// Wide lm head over the final row of each request (apply_head lm_logits, model.cpp:151-168):
// gather (+ f64 LayerNorm of pre-norm rows), tcgen05 logits GEMM, top-8 + f64 rescoring.
void Ctx::launch_lm_head(uint32_t n_req, int S, const LmHead& lm, int wide_head, bool gen,
                         float* scores, int32_t* labels) {
  cudaStream_t s = compute;
  const int prec = static_cast<int>(opt.precision);
  const int Mp = static_cast<int>((n_req + 127) / 128 * 128);
  launch_lm_gather(h16.p, h32.p, layers[L - 1].ln2g, layers[L - 1].ln2b,
                   d_lens.p, static_cast<int>(n_req), S, d, prec, hdec32.p, hdec16.p, s);
  launch_gemm(lm.plan, Mp, s);
  LmArgmaxArgs a;
  a.logits = lm_logits.p;
  a.ld = static_cast<int>(lm_logits.n / Bp);
  a.V = lm.V;
  a.h32 = hdec32.p;
  a.d = d;
  a.w = d_head_arena.p + h_head_off[wide_head];
  a.bias = a.w + static_cast<size_t>(d) * lm.V;
  a.wT = lm.wT;
  if (gen) {
    // the prompt's tokens start the generated sequences; token 1 lands at position len
    HMI_CUDA(cudaMemcpy2DAsync(gen_tokens.p, static_cast<size_t>(gen_stride) * 4, d_tokens.p,
                               static_cast<size_t>(S) * 4, static_cast<size_t>(S) * 4, n_req,
                               cudaMemcpyDeviceToDevice, s));
    HMI_CUDA(cudaMemcpyAsync(gen_pos.p, d_lens.p, n_req * 4, cudaMemcpyDeviceToDevice, s));
    a.gen_tokens = gen_tokens.p;
    a.tok_stride = gen_stride;
    a.gen_pos = gen_pos.p;
    a.advance = 0;
    a.out_tokens = gen_out.p;
    a.out_logits = gen_logit.p;
    a.out_ld = static_cast<int>(opt.max_new_tokens);
    a.step = 0;
  } else {
    a.req_head = d_req_head.p;
    a.head = wide_head;
    a.labels_out = labels;
    a.scores_out = scores;
    a.scores_ld = static_cast<int>(opt.max_labels);
  }
  launch_lm_argmax(a, static_cast<int>(n_req), s);
}

// Generated tokens 2..n_new: one causal row per request per step through every layer,
// keys / values of earlier rows read from the cache (prompt rows: qkv_at(l); generated
// rows: kv_tail). Each step: K5 (decode row) -> per layer QKV, cached attention, O,
// per-row adapter + LN1, FFN1, FFN2 (+res), LN2 -> lm GEMM -> argmax / append.
void Ctx::decode_steps(uint32_t n_req, uint32_t n_new, int S, const LmHead& lm, int wide_head) {
  cudaStream_t s = compute;
  const int prec = static_cast<int>(opt.precision);
  const int n = static_cast<int>(n_req);
  const int Mp = (n + 127) / 128 * 128;
  const int T = static_cast<int>(opt.max_new_tokens);
  PlotDev P;
  P.slots = d_slots.p;
  P.mask = h_slots.empty() ? 0 : h_slots.size() - 1;
  P.parent = d_parent.p;
  P.max_versions = static_cast<int>(h_parent.size());
  P.reps = d_reps.p;
  P.ngram = ngram;
  P.d = d;
  P.max_depth = 1;
  for (size_t v = 0; v < h_parent.size(); ++v) {
    if (h_parent[v] == -2) continue;
    int depth = 1;
    for (int32_t u = h_parent[v]; u >= 0; u = h_parent[u]) ++depth;
    P.max_depth = std::max(P.max_depth, depth);
  }
  LmArgmaxArgs am;
  am.logits = lm_logits.p;
  am.ld = static_cast<int>(lm_logits.n / Bp);
  am.V = lm.V;
  am.h32 = hdec32.p;
  am.d = d;
  am.w = d_head_arena.p + h_head_off[wide_head];
  am.wT = lm.wT;
  am.bias = am.w + static_cast<size_t>(d) * lm.V;
  am.gen_tokens = gen_tokens.p;
  am.tok_stride = gen_stride;
  am.gen_pos = gen_pos.p;
  am.advance = 1;
  am.out_tokens = gen_out.p;
  am.out_logits = gen_logit.p;
  am.out_ld = T;
  auto launch_dec = [&](const DecGemmPlan& kp, const GemmPlan& g) {
    if (kp.fn) {
      launch_dec_gemm(kp, Mp, s);
    } else {
      launch_gemm(g, Mp, s);
    }
  };
  auto step = [&](uint32_t k) {
    timed(P_RETRIEVE, s, [&] {
      launch_retrieve(P, gen_tokens.p, d_lens.p, d_req_version.p, n, S, 1, h16.p, prec, nullptr,
                      nullptr, nullptr, d_err.p, s, gen_pos.p, gen_stride);
    });
    for (int l = 0; l < L; ++l) {
      LayerDev& w = layers[l];
      DecPlans& dp = dec[l];
      const bool last = l == L - 1;
      timed(P_QKV, s, [&] { launch_dec(dp.kqkv, dp.qkv); });
      timed(P_ATTN, s, [&] {
        AttnDecodeArgs a;
        a.qkv_new = qkv_dec.p;
        a.qkv_prefill = qkv_at(l);
        a.S = S;
        a.tail = kv_tail.p + static_cast<size_t>(l) * opt.max_batch * T * 2 * d;
        a.tail_cap = T;
        a.lens = d_lens.p;
        a.gen_pos = gen_pos.p;
        a.ctx = ctx16.p;
        a.d = d;
        a.scale = static_cast<float>(1.0 / std::sqrt(static_cast<double>(d / heads)));
        a.bf16 = prec;
        if (attn_decode_tma_ok(S, T)) {
          launch_attn_decode_tma(a, dec[l].attn, n, heads, s);
        } else {
          launch_attn_decode(a, n, heads, S + static_cast<int>(n_new), s);
        }
      });
      timed(P_OPROJ, s, [&] { launch_dec(dp.koproj, dp.oproj); });
      timed(P_AD_UP, s, [&] {
        AdapterRowsArgs a;
        a.ctx16 = ctx16.p;
        a.a16 = a16.p;
        a.h16 = h16.p;
        a.req_task = d_req_task.p;
        a.slot_of = d_slot_of.p;
        a.layers = L;
        a.layer = l;
        a.arena = arena.p;
        a.slot_bytes = slot_bytes;
        a.d = d;
        a.r_pad = r_pad;
        a.ln_g = w.ln1g;
        a.ln_b = w.ln1b;
        a.x16 = x16.p;
        a.err = d_err.p;
        a.bf16 = prec;
        launch_adapter_rows_ln(a, n, s);
      });
      timed(P_FFN1, s, [&] { launch_dec(dp.kffn1, dp.ffn1); });
      timed(P_FFN2, s, [&] { launch_dec(dp.kffn2, dp.ffn2); });
      timed(P_LN2, s, [&] {
        launch_layernorm(y32.p, w.ln2g, w.ln2b, last ? hdec16.p : h16.p, last ? hdec32.p : nullptr,
                         n, d, prec, s);
      });
    }
    timed(P_HEAD, s, [&] {
      launch_gemm(lm.plan, Mp, s);
      (void)k;
      am.step = -1;  // output column from gen_pos: identical launches every step
      am.lens = d_lens.p;
      launch_lm_argmax(am, n, s);
    });
  };
  // step 1 eagerly (first-use attribute setup), then one captured step replayed: a decode step
  // is ~90 short launches whose arguments do not change between steps (positions live on the
  // device), so the graph removes the per-launch submission and inter-kernel gaps
  if (n_new <= 1) return;
  step(1);
  // debug flag 4 (hmi_gpu_set_debug): eager launches every step (tests compare the two)
  const bool graph = !(debug_flags & 4) && !prof && n_new > 2;
  if (!graph) {
    for (uint32_t k = 2; k < n_new; ++k) step(k);
    return;
  }
  const auto key = std::make_tuple(n, S, wide_head, tables_epoch);
  for (auto g = dec_graphs.begin(); g != dec_graphs.end();) {  // graphs of replaced table state
    if (std::get<3>(g->first) != tables_epoch) {
      HMI_CUDA(cudaStreamSynchronize(s));
      cudaGraphExecDestroy(g->second);
      g = dec_graphs.erase(g);
    } else {
      ++g;
    }
  }
  auto it = dec_graphs.find(key);
  if (it == dec_graphs.end()) {
    cudaGraph_t g = nullptr;
    HMI_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    step(2);
    HMI_CUDA(cudaStreamEndCapture(s, &g));
    cudaGraphExec_t exec = nullptr;
    const cudaError_t e = cudaGraphInstantiate(&exec, g, 0);
    cudaGraphDestroy(g);
    HMI_CUDA(e);
    it = dec_graphs.emplace(key, exec).first;
  }
  for (uint32_t k = 2; k < n_new; ++k) HMI_CUDA(cudaGraphLaunch(it->second, s));
}

}  // namespace hmi_b200

// ===========================================================================
// C ABI
// ===========================================================================
using hmi_b200::Ctx;
using hmi_b200::HmiError;

struct hmi_gpu_ctx {
  Ctx impl;
};

namespace {

template <typename F>
int guarded(F&& fn) {
  try {
    fn();
    return HMI_OK;
  } catch (const HmiError& e) {
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

// ModelConfig::validate (weights.cpp:56-70) plus the device constraints.
void validate(const hmi_model_config& c, const hmi_gpu_options& o) {
  if (c.hidden_size == 0 || c.heads == 0 || c.hidden_size % c.heads != 0)
    throw HmiError(HMI_CONFIG_ERROR, "hidden_size must be a positive multiple of heads");
  if (c.lower_layers < 1 || c.higher_layers < 1)
    throw HmiError(HMI_CONFIG_ERROR, "lower_layers and higher_layers must both be >= 1");
  if (c.ffn_size == 0 || c.vocab_size == 0)
    throw HmiError(HMI_CONFIG_ERROR, "ffn_size and vocab_size must be positive");
  if (c.max_fragment != 1 && c.max_fragment != 2 && c.max_fragment != 3 && c.max_fragment != 5)
    throw HmiError(HMI_CONFIG_ERROR, "max_fragment must be one of {1, 2, 3, 5}");
  if (c.hidden_size / c.heads != 64)
    throw HmiError(HMI_CONFIG_ERROR, "device path requires hidden_size / heads == 64");
  if (c.hidden_size % 128 != 0 || c.ffn_size % 64 != 0)
    throw HmiError(HMI_CONFIG_ERROR, "device path requires hidden_size % 128 == 0 and ffn % 64 == 0");
  if (o.bottleneck == 0 || o.bottleneck >= c.hidden_size || o.bottleneck > 256)
    throw HmiError(HMI_CONFIG_ERROR, "adapter bottleneck must be in [1, min(hidden_size, 257))");
  if (o.max_batch == 0 || o.max_seq == 0 || o.max_labels == 0)
    throw HmiError(HMI_CONFIG_ERROR, "max_batch, max_seq and max_labels must be positive");
  if (o.precision > 1) throw HmiError(HMI_CONFIG_ERROR, "precision must be 0 (fp16) or 1 (bf16)");
  if (o.pipeline_mode > 2) throw HmiError(HMI_CONFIG_ERROR, "pipeline_mode must be 0, 1 or 2");
  if (c.vocab_size >= (1u << 31)) throw HmiError(HMI_CONFIG_ERROR, "vocab too large");
}

}  // namespace

extern "C" {

int hmi_gpu_create(int device, const hmi_model_config* cfg, const hmi_gpu_options* opts,
                   const float* higher_f32, hmi_gpu_ctx** out) {
  using namespace hmi_b200;
  *out = nullptr;
  auto holder = std::make_unique<hmi_gpu_ctx>();
  int rc = guarded([&] {
    HMI_CHECK(cfg && opts && higher_f32, HMI_CONFIG_ERROR, "null argument");
    validate(*cfg, *opts);
    Ctx& c = holder->impl;
    c.device = device;
    c.cfg = *cfg;
    c.opt = *opts;
    if (c.opt.max_tasks == 0) c.opt.max_tasks = 1024;
    if (c.opt.max_instances == 0) c.opt.max_instances = c.opt.max_tasks;
    if (c.opt.max_heads == 0) c.opt.max_heads = c.opt.max_tasks;
    if (c.opt.max_versions == 0) c.opt.max_versions = 64;
    HMI_CUDA(cudaSetDevice(device));
    c.numa_node = gpu_numa_node(device);
    c.d = static_cast<int>(cfg->hidden_size);
    c.f = static_cast<int>(cfg->ffn_size);
    c.L = static_cast<int>(cfg->higher_layers);
    c.heads = static_cast<int>(cfg->heads);
    c.ngram = static_cast<int>(cfg->max_fragment);
    c.r = static_cast<int>(opts->bottleneck);
    c.r_pad = (c.r + 63) / 64 * 64;
    c.S_max = static_cast<int>((opts->max_seq + 127) / 128 * 128);
    c.max_rows = static_cast<int>(c.opt.max_batch) * c.S_max;
    c.tile_stride = c.max_rows / 128;
    c.slot_bytes = (static_cast<size_t>(c.r_pad) * c.d * 2 * 2 + (c.r_pad + c.d) * 4 + 1023) / 1024 * 1024;
    c.ref_layer_bytes = (static_cast<uint64_t>(c.d) * c.r * 2 + c.r + c.d) * 4;
    HMI_CUDA(cudaStreamCreateWithFlags(&c.compute, cudaStreamNonBlocking));
    HMI_CUDA(cudaStreamCreateWithFlags(&c.copy, cudaStreamNonBlocking));
    HMI_CUDA(cudaStreamCreateWithFlags(&c.copy2, cudaStreamNonBlocking));
    HMI_CUDA(cudaEventCreateWithFlags(&c.ev_fork, cudaEventDisableTiming));
    HMI_CUDA(cudaEventCreateWithFlags(&c.ev_join, cudaEventDisableTiming));
    c.ev_layer.resize(c.L);
    for (auto& e : c.ev_layer) HMI_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    c.d_ready.alloc(c.L);
    HMI_CUDA(cudaMemset(c.d_ready.p, 0, c.L * sizeof(uint32_t)));
    c.write_value32 = stream_write_value32();

    // ---- shared weights: [in x out] f32 -> [out][in] 16-bit, biases / LN f32
    const size_t d = c.d, f = c.f;
    const size_t lf = 4 * (d * d + d) + (d * f + f) + (f * d + d) + 4 * d;
    const int prec = static_cast<int>(c.opt.precision);
    c.layers.resize(c.L);
    c.wo32.alloc(static_cast<size_t>(c.L) * d * d);
    c.bo32.alloc(static_cast<size_t>(c.L) * d);
    std::vector<uint16_t> tmp;
    for (int l = 0; l < c.L; ++l) {
      const float* w = higher_f32 + l * lf;
      const float *wq = w, *bq = wq + d * d, *wk = bq + d, *bk = wk + d * d, *wv = bk + d,
                  *bv = wv + d * d, *wo = bv + d, *bo = wo + d * d, *w1 = bo + d, *b1 = w1 + d * f,
                  *w2 = b1 + f, *b2 = w2 + f * d, *g1 = b2 + d, *s1 = g1 + d, *g2 = s1 + d,
                  *s2 = g2 + d;
      const size_t n16 = 3 * d * d + d * d + f * d + d * f;
      const size_t n32 = 3 * d + d + f + d + 4 * d;
      LayerDev& L = c.layers[l];
      HMI_CUDA(cudaMalloc(&L.mem, n16 * 2 + n32 * 4 + 1024));
      uint16_t* p16 = static_cast<uint16_t*>(L.mem);
      L.wqkv = p16; L.wo = L.wqkv + 3 * d * d; L.w1 = L.wo + d * d; L.w2 = L.w1 + f * d;
      float* p32 = reinterpret_cast<float*>(L.w2 + d * f);
      L.bqkv = p32; L.bo = L.bqkv + 3 * d; L.b1 = L.bo + d; L.b2 = L.b1 + f;
      L.ln1g = L.b2 + d; L.ln1b = L.ln1g + d; L.ln2g = L.ln1b + d; L.ln2b = L.ln2g + d;
      tmp.assign(n16, 0);
      auto transpose = [&](const float* src, size_t in, size_t outn, uint16_t* dst) {
        for (size_t o = 0; o < outn; ++o)
          for (size_t i = 0; i < in; ++i) dst[o * in + i] = f2h(src[i * outn + o], prec);
      };
      transpose(wq, d, d, tmp.data());
      transpose(wk, d, d, tmp.data() + d * d);
      transpose(wv, d, d, tmp.data() + 2 * d * d);
      transpose(wo, d, d, tmp.data() + 3 * d * d);
      HMI_CUDA(cudaMemcpy(c.wo32.p + l * d * d, wo, d * d * 4, cudaMemcpyHostToDevice));
      HMI_CUDA(cudaMemcpy(c.bo32.p + l * d, bo, d * 4, cudaMemcpyHostToDevice));
      transpose(w1, d, f, tmp.data() + 4 * d * d);
      transpose(w2, f, d, tmp.data() + 4 * d * d + f * d);
      HMI_CUDA(cudaMemcpy(p16, tmp.data(), n16 * 2, cudaMemcpyHostToDevice));
      std::vector<float> v32;
      v32.insert(v32.end(), bq, bq + d);
      v32.insert(v32.end(), bk, bk + d);
      v32.insert(v32.end(), bv, bv + d);
      v32.insert(v32.end(), bo, bo + d);
      v32.insert(v32.end(), b1, b1 + f);
      v32.insert(v32.end(), b2, b2 + d);
      v32.insert(v32.end(), g1, g1 + d);
      v32.insert(v32.end(), s1, s1 + d);
      v32.insert(v32.end(), g2, g2 + d);
      v32.insert(v32.end(), s2, s2 + d);
      HMI_CUDA(cudaMemcpy(p32, v32.data(), v32.size() * 4, cudaMemcpyHostToDevice));
      // LN folding: FFN1 consumes pre-LN1 y1 (this layer's LN1); QKV of layer l >= 1
      // consumes pre-LN2 y2 of layer l-1 (that layer's LN2)
      {
        std::vector<uint16_t> wf1, wfq, tmpq;
        std::vector<float> bf1, cs1, bfq, csq;
        fold_weights(w1, d, f, b1, g1, s1, prec, wf1, bf1, cs1);
        const size_t bytes = (3 * d * d + f * d) * 2 + (2 * 3 * d + 2 * f) * 4 + 1024;
        HMI_CUDA(cudaMalloc(&L.mem_fold, bytes));
        uint16_t* f16p = static_cast<uint16_t*>(L.mem_fold);
        L.wqkv_f = f16p;
        L.w1_f = f16p + 3 * d * d;
        float* f32p = reinterpret_cast<float*>(L.w1_f + f * d);
        L.bqkv_f = f32p;
        L.cs_qkv = f32p + 3 * d;
        L.b1_f = f32p + 6 * d;
        L.cs_1 = f32p + 6 * d + f;
        HMI_CUDA(cudaMemcpy(L.w1_f, wf1.data(), wf1.size() * 2, cudaMemcpyHostToDevice));
        HMI_CUDA(cudaMemcpy(L.b1_f, bf1.data(), f * 4, cudaMemcpyHostToDevice));
        HMI_CUDA(cudaMemcpy(L.cs_1, cs1.data(), f * 4, cudaMemcpyHostToDevice));
        if (l > 0) {
          const float* pw = higher_f32 + (l - 1) * lf;
          const float* pg2 = pw + 4 * (d * d + d) + (d * f + f) + (f * d + d) + 2 * d;
          const float* ps2 = pg2 + d;
          // concatenated [wq | wk | wv] as one [d][3d] matrix, biases [bq | bk | bv]
          std::vector<float> wcat(d * 3 * d), bcat(3 * d);
          for (size_t i = 0; i < d; ++i)
            for (size_t o = 0; o < d; ++o) {
              wcat[i * 3 * d + o] = wq[i * d + o];
              wcat[i * 3 * d + d + o] = wk[i * d + o];
              wcat[i * 3 * d + 2 * d + o] = wv[i * d + o];
            }
          for (size_t o = 0; o < d; ++o) {
            bcat[o] = bq[o];
            bcat[d + o] = bk[o];
            bcat[2 * d + o] = bv[o];
          }
          fold_weights(wcat.data(), d, 3 * d, bcat.data(), pg2, ps2, prec, wfq, bfq, csq);
          HMI_CUDA(cudaMemcpy(L.wqkv_f, wfq.data(), wfq.size() * 2, cudaMemcpyHostToDevice));
          HMI_CUDA(cudaMemcpy(L.bqkv_f, bfq.data(), 3 * d * 4, cudaMemcpyHostToDevice));
          HMI_CUDA(cudaMemcpy(L.cs_qkv, csq.data(), 3 * d * 4, cudaMemcpyHostToDevice));
        }
      }
    }

    // ---- activations
    const size_t R = c.max_rows;
    c.kv = c.opt.max_new_tokens > 0;
    HMI_CHECK(!c.kv || cfg->mode == 1, HMI_CONFIG_ERROR,
              "max_new_tokens needs a causal model (encoder rows see later tokens)");
    c.Bp = static_cast<int>((c.opt.max_batch + 127) / 128 * 128);
    c.h16.alloc(R * d); c.qkv16.alloc(R * 3 * d * (c.kv ? c.L : 1)); c.ctx16.alloc(R * d); c.a16.alloc(R * d);
    c.hdec16.alloc(static_cast<size_t>(c.Bp) * d);
    c.hdec32.alloc(static_cast<size_t>(c.Bp) * d);
    if (c.kv) {
      const size_t Bm = c.opt.max_batch, T = c.opt.max_new_tokens;
      c.qkv_dec.alloc(static_cast<size_t>(c.Bp) * 3 * d);
      c.kv_tail.alloc(static_cast<size_t>(c.L) * Bm * T * 2 * d);
      c.gen_stride = c.S_max + static_cast<int>(T);
      c.gen_tokens.alloc(Bm * c.gen_stride);
      c.gen_pos.alloc(Bm);
      c.gen_out.alloc(Bm * T);
      c.gen_logit.alloc(Bm * T);
    }
    // + 128 zero rows: the other CTA's half of the O projection's tenant K blocks
    c.mid16.alloc((R + 128) * c.r_pad);
    HMI_CUDA(cudaMemset(c.mid16.p, 0, c.mid16.n * 2)); c.x16.alloc(R * d); c.ffn16.alloc(R * f);
    c.y32.alloc(R * d); c.h32.alloc(R * d);
    const size_t B = c.opt.max_batch;
    c.d_inst.alloc(B); c.d_tokens.alloc(B * c.S_max); c.d_lens.alloc(B);
    c.d_req_version.alloc(B); c.d_req_task.alloc(B); c.d_req_head.alloc(B);
    c.d_tile_slot.alloc(static_cast<size_t>(c.L) * c.tile_stride);
    HMI_CUDA(cudaMemset(c.d_tile_slot.p, 0, c.d_tile_slot.n * 4));
    c.d_err.alloc(1);
    c.d_gather.alloc(R * c.ngram); c.d_levels.alloc(R * c.ngram);
    c.d_scores.alloc(B * c.opt.max_labels); c.d_labels.alloc(B); c.d_tags.alloc(R);
    const size_t max_delta = B * c.L * (c.L + 2) + 64;
    c.d_delta.alloc(2 * max_delta);
    for (auto& s : c.stg) {
      HMI_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&s.inst), B * 4, 0));
      HMI_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&s.tokens), B * c.S_max * 4, 0));
      HMI_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&s.lens), B * 4, 0));
      HMI_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&s.delta), 2 * max_delta * 4, 0));
      HMI_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&s.scores), B * c.opt.max_labels * 4, 0));
      HMI_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&s.labels), B * 4, 0));
      HMI_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&s.tags), R * 4, 0));
      HMI_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&s.err), 4, 0));
      HMI_CUDA(cudaEventCreateWithFlags(&s.done, cudaEventDisableTiming));
    }

    // ---- routing tables
    c.h_inst_version.assign(c.opt.max_instances, -1);
    c.h_inst_task.assign(c.opt.max_instances, -1);
    c.h_inst_head.assign(c.opt.max_instances, -1);
    c.d_inst_version.alloc(c.opt.max_instances);
    c.d_inst_task.alloc(c.opt.max_instances);
    c.d_inst_head.alloc(c.opt.max_instances);
    HMI_CUDA(cudaMemset(c.d_inst_version.p, 0xff, c.opt.max_instances * 4));
    HMI_CUDA(cudaMemset(c.d_inst_task.p, 0xff, c.opt.max_instances * 4));
    HMI_CUDA(cudaMemset(c.d_inst_head.p, 0xff, c.opt.max_instances * 4));
    c.d_slot_of.alloc(static_cast<size_t>(c.opt.max_tasks) * c.L);
    HMI_CUDA(cudaMemset(c.d_slot_of.p, 0xff, c.d_slot_of.n * 4));
    c.store.assign(c.opt.max_tasks, nullptr);

    // ---- heads
    c.h_head_off.assign(c.opt.max_heads, -1);
    c.h_head_labels.assign(c.opt.max_heads, 0);
    c.h_head_kind.assign(c.opt.max_heads, -1);
    c.d_head_off.alloc(c.opt.max_heads);
    c.d_head_labels.alloc(c.opt.max_heads);
    c.d_head_kind.alloc(c.opt.max_heads);
    HMI_CUDA(cudaMemset(c.d_head_off.p, 0, c.opt.max_heads * 8));
    HMI_CUDA(cudaMemset(c.d_head_labels.p, 0, c.opt.max_heads * 4));
    HMI_CUDA(cudaMemset(c.d_head_kind.p, 0, c.opt.max_heads * 4));

    // ---- PLOT
    c.h_parent.assign(c.opt.max_versions, -2);
    c.d_parent.alloc(c.opt.max_versions);
    c.h_slots.assign(1024, PlotSlot{kEmptyKey, 0, {0, 0, 0, 0, 0}, 0});

    // ---- adapter slot pool: HBM arena sized by the byte budget
    uint64_t pool_bytes = c.opt.pool_bytes;
    if (pool_bytes == 0) pool_bytes = static_cast<uint64_t>(c.opt.max_tasks) * c.L * c.ref_layer_bytes;
    uint64_t n_slots64 = pool_bytes / c.ref_layer_bytes;
    HMI_CHECK(n_slots64 >= 1 && n_slots64 < (1ull << 31), HMI_CONFIG_ERROR,
              "pool_bytes must hold at least one adapter layer");
    // physical placement headroom: one spare block of L slots per request of a batch, so a
    // whole-task miss finds a free block (contiguous copy) even while the byte budget is full
    // and the budget frees slots one evicted task at a time (slot_pool.hpp); residency is
    // still decided by the byte budget alone
    const uint64_t n_phys = n_slots64 / c.L * c.L + static_cast<uint64_t>(c.L) * c.opt.max_batch;
    HMI_CHECK(n_phys < (1ull << 31), HMI_CONFIG_ERROR, "pool_bytes too large");
    n_slots64 = n_phys;
    c.pool = std::make_unique<SlotPool>(pool_bytes, static_cast<uint32_t>(n_slots64),
                                        static_cast<uint32_t>(c.L));
    c.arena.alloc(static_cast<size_t>(n_slots64) * c.slot_bytes);
    HMI_CUDA(cudaMemset(c.arena.p, 0, c.arena.n));
    c.oproj_ext = c.r_pad == 64 && c.d % 128 == 0;
    c.d_stats1.alloc(static_cast<size_t>(c.max_rows) * Ctx::kStatsLd);
    c.d_stats2.alloc(static_cast<size_t>(c.max_rows) * Ctx::kStatsLd);
    c.build_plans();
    HMI_CUDA(cudaDeviceSynchronize());
  });
  if (rc == HMI_OK) *out = holder.release();
  return rc;
}

int hmi_gpu_destroy(hmi_gpu_ctx* ctx) {
  if (!ctx) return HMI_OK;
  cudaSetDevice(ctx->impl.device);
  delete ctx;
  return HMI_OK;
}

namespace hmi_b200 {
// VersionTree::add_branch checks (version_tree.cpp): free id, existing parent, one root, depth.
static void check_new_version(Ctx& c, uint32_t version_id, uint32_t parent_id) {
  HMI_CHECK(version_id < c.h_parent.size(), HMI_CONFIG_ERROR, "version id exceeds max_versions");
  if (c.h_parent[version_id] != -2) throw HmiError(HMI_CONFLICT_ERROR, "version already exists");
  if (parent_id != kNoParent) {
    if (parent_id >= c.h_parent.size() || c.h_parent[parent_id] == -2)
      throw HmiError(HMI_ROUTING_ERROR, "branch parent version " + std::to_string(parent_id) +
                                            " does not exist");
    int depth = 2;  // device retrieval resolves chains of up to 8 tables
    for (int32_t v = c.h_parent[parent_id]; v >= 0; v = c.h_parent[v]) ++depth;
    HMI_CHECK(depth <= 8, HMI_CONFIG_ERROR, "version tree deeper than 8 levels");
  } else {
    for (int32_t p : c.h_parent)
      if (p == -1) throw HmiError(HMI_CONFLICT_ERROR, "a root table is already registered");
  }
}

// Keys of one version into a copy of the host hash (fail-closed on duplicates); returns it with
// the hash grown to keep load <= 0.5. Rows are numbered from c.rep_rows on.
static std::vector<PlotSlot> stage_keys(Ctx& c, uint32_t version_id, uint32_t n_entries,
                                        const uint32_t* key_len, const uint32_t* keys,
                                        uint64_t* rows_out) {
  const uint32_t n = static_cast<uint32_t>(c.ngram);
  uint64_t rows = 0;
  for (uint32_t e = 0; e < n_entries; ++e) {
    if (key_len[e] == 0 || key_len[e] > n)
      throw HmiError(HMI_FORMAT_ERROR, "entry key length outside [1, n]");
    for (uint32_t j = 0; j < key_len[e]; ++j)
      if (keys[static_cast<size_t>(e) * n + j] >= c.cfg.vocab_size)
        throw HmiError(HMI_VOCABULARY_ERROR, "key token outside vocabulary");
    rows += key_len[e];
  }
  uint64_t need = c.n_keys + n_entries;
  if (need * 2 > c.h_slots.size()) {
    uint64_t cap = c.h_slots.size();
    while (need * 2 > cap) cap <<= 1;
    std::vector<PlotSlot> old;
    old.swap(c.h_slots);
    c.h_slots.assign(cap, PlotSlot{kEmptyKey, 0, {0, 0, 0, 0, 0}, 0});
    for (const PlotSlot& s : old) {
      if (s.version == kEmptyKey) continue;
      uint64_t i = plot_hash(s.version, s.len, s.tok) & (cap - 1);
      while (c.h_slots[i].version != kEmptyKey) i = (i + 1) & (cap - 1);
      c.h_slots[i] = s;
    }
  }
  std::vector<PlotSlot> staged(c.h_slots);
  const uint64_t mask = staged.size() - 1;
  uint64_t row = c.rep_rows;
  for (uint32_t e = 0; e < n_entries; ++e) {
    PlotSlot s{version_id, key_len[e], {0, 0, 0, 0, 0}, static_cast<uint32_t>(row)};
    for (uint32_t j = 0; j < key_len[e]; ++j) s.tok[j] = keys[static_cast<size_t>(e) * n + j];
    uint64_t i = plot_hash(s.version, s.len, s.tok) & mask;
    for (;; i = (i + 1) & mask) {
      const PlotSlot& o = staged[i];
      if (o.version == kEmptyKey) break;
      if (o.version == s.version && o.len == s.len &&
          std::memcmp(o.tok, s.tok, sizeof(uint32_t) * s.len) == 0)
        throw HmiError(HMI_FORMAT_ERROR, "duplicate entry key");
    }
    staged[i] = s;
    row += key_len[e];
  }
  HMI_CHECK(row < (1ull << 31), HMI_CAPACITY_ERROR, "PLOT row count exceeds 2^31");
  *rows_out = rows;
  return staged;
}

// pread of [off, off + n) into dst by up to 4 threads; returns the bytes read.
static size_t read_parallel(int fd, uint8_t* dst, size_t n, uint64_t off) {
  if (n == 0) return 0;
  const int parts = n >= (size_t(8) << 20) ? 4 : 1;
  const size_t step = (n + parts - 1) / parts;
  size_t got[4] = {0, 0, 0, 0};
  auto work = [&](int i) {
    const size_t a = i * step, b = std::min(n, a + step);
    size_t done = 0;
    while (a + done < b) {
      const ssize_t r = pread(fd, dst + a + done, b - a - done, static_cast<off_t>(off + a + done));
      if (r <= 0) break;
      done += static_cast<size_t>(r);
    }
    got[i] = done;
  };
  std::vector<std::thread> th;
  for (int i = 1; i < parts; ++i) th.emplace_back(work, i);
  work(0);
  for (auto& t : th) t.join();
  size_t total = 0;
  for (int i = 0; i < parts; ++i) total += got[i];
  return total;
}

// The reps arena holds at least `rows` rows (appending, growing geometrically).
static void reserve_rep_rows(Ctx& c, uint64_t rows) {
  const size_t need_f = static_cast<size_t>(rows) * c.d;
  if (need_f <= c.d_reps.n) return;
  c.drop_decode_graphs();
  DevBuf<float> grown;
  grown.alloc(std::max(need_f, c.d_reps.n * 3 / 2 + 1));
  if (c.rep_rows) HMI_CUDA(cudaMemcpy(grown.p, c.d_reps.p, c.rep_rows * c.d * 4, cudaMemcpyDeviceToDevice));
  c.d_reps.free();
  c.d_reps = grown;
  grown.p = nullptr;
}

static void commit_version(Ctx& c, uint32_t version_id, uint32_t parent_id, uint32_t n_entries,
                           uint64_t rows, std::vector<PlotSlot>& staged) {
  c.h_slots.swap(staged);
  c.n_keys += n_entries;
  c.rep_rows += rows;
  c.h_parent[version_id] = parent_id == kNoParent ? -1 : static_cast<int32_t>(parent_id);
  c.upload_plot_hash();
  c.drop_decode_graphs();  // retrieval pointers / hash mask may have changed: recapture
  ++c.tables_epoch;
}
}  // namespace hmi_b200

int hmi_gpu_upload_table(hmi_gpu_ctx* ctx, uint32_t version_id, uint32_t parent_id,
                         uint32_t n_entries, const uint32_t* key_len, const uint32_t* keys,
                         const float* reps) {
  using namespace hmi_b200;
  return guarded([&] {
    Ctx& c = ctx->impl;
    std::lock_guard<std::mutex> lock(c.mu);
    HMI_CUDA(cudaSetDevice(c.device));
    c.reap(true);
    check_new_version(c, version_id, parent_id);
    uint64_t rows = 0;
    auto staged = stage_keys(c, version_id, n_entries, key_len, keys, &rows);
    reserve_rep_rows(c, c.rep_rows + rows);
    if (rows)
      HMI_CUDA(cudaMemcpy(c.d_reps.p + c.rep_rows * c.d, reps, rows * c.d * 4, cudaMemcpyHostToDevice));
    commit_version(c, version_id, parent_id, n_entries, rows, staged);
  });
}

// Streaming PLT1 ingest (plot_io.cpp:35-72 format): the file is read in chunks straight into
// pinned memory and each chunk goes to the GPU whole; a kernel moves the entries' rep rows out
// of the raw chunk into the reps arena while the host reads the next chunk. The host touches
// only the entry headers; validation and fail-closed commit as hmi_gpu_upload_table.
int hmi_gpu_upload_plt1(hmi_gpu_ctx* ctx, const char* path, uint32_t* version_out,
                        uint32_t* parent_out) {
  using namespace hmi_b200;
  return guarded([&] {
    HMI_CHECK(ctx != nullptr && path != nullptr, HMI_CONFIG_ERROR, "null argument");
    Ctx& c = ctx->impl;
    std::lock_guard<std::mutex> lock(c.mu);
    HMI_CUDA(cudaSetDevice(c.device));
    c.reap(true);
    FILE* f = std::fopen(path, "rb");
    if (!f) throw HmiError(HMI_FORMAT_ERROR, std::string("cannot open ") + path + " (offset 0)");
    struct Closer {
      FILE* f;
      ~Closer() { std::fclose(f); }
    } closer{f};
    std::fseek(f, 0, SEEK_END);
    const uint64_t file_size = static_cast<uint64_t>(std::max<long>(0, std::ftell(f)));
    std::fseek(f, 0, SEEK_SET);
    auto fail = [](const std::string& what, uint64_t at) {
      throw HmiError(HMI_FORMAT_ERROR, what + " (offset " + std::to_string(at) + ")");
    };
    // header (small, plain reads)
    uint64_t off = 0;
    auto rd = [&](void* p, size_t n) {
      if (off + n > file_size || std::fread(p, 1, n, f) != n) fail("unexpected end of file", off);
      off += n;
    };
    char magic[4];
    rd(magic, 4);
    if (std::memcmp(magic, "PLT1", 4) != 0) fail("bad magic, expected PLT1", 0);
    uint32_t version = 0, parent = 0, label_len = 0, ngram = 0, d = 0, count = 0, alpha = 0;
    rd(&version, 4);
    rd(&parent, 4);
    const uint64_t label_at = off;
    rd(&label_len, 4);
    if (label_len > (1u << 20)) fail("string length " + std::to_string(label_len) + " implausible", label_at);
    std::vector<char> label(label_len);
    if (label_len) rd(label.data(), label_len);
    rd(&ngram, 4);
    rd(&d, 4);
    rd(&count, 4);
    rd(&alpha, 4);
    if (ngram == 0 || d == 0) fail("table header has zero ngram or hidden size", off);
    HMI_CHECK(ngram == static_cast<uint32_t>(c.ngram) && d == static_cast<uint32_t>(c.d),
              HMI_DIMENSION_ERROR, "PLT1 table (ngram " + std::to_string(ngram) + ", d " +
                                       std::to_string(d) + ") does not match the model");
    // the tree checks (free id, existing parent) come after the whole file parsed, as the
    // reference's load() then VersionTree::add_branch: a truncated file is a FormatError first
    const bool dbg = std::getenv("HMI_DEBUG_INGEST") != nullptr;
    auto now = [] { return std::chrono::duration<double, std::milli>(
                        std::chrono::steady_clock::now().time_since_epoch()).count(); };
    double t_a = now(), t_read = 0, t_parse = 0, t_wait = 0;
    // rows are bounded by the payload size: reserve once, stream into [rep_rows, ...)
    const uint64_t row_bytes = static_cast<uint64_t>(d) * 4;
    reserve_rep_rows(c, c.rep_rows + (file_size - off) / row_bytes + 1);
    float* dst_base = c.d_reps.p + c.rep_rows * c.d;

    const size_t kChunk = size_t(64) << 20;
    const size_t max_entry = 4 + 4 * ngram + 8 + ngram * row_bytes;
    HMI_CHECK(max_entry <= kChunk, HMI_CONFIG_ERROR, "PLT1 entry larger than the ingest chunk");
    struct Slot {
      uint8_t* host = nullptr;
      int4* segs_h = nullptr;  // {src byte offset in chunk, dst row (low), dst row (high), rows}
      uint8_t* dev = nullptr;
      int4* segs_d = nullptr;
      cudaEvent_t done = nullptr;
      size_t seg_cap = 0;
    } slot[2];
    struct Freer {
      Slot* s;
      ~Freer() {
        for (int i = 0; i < 2; ++i) {
          if (s[i].done) cudaEventSynchronize(s[i].done), cudaEventDestroy(s[i].done);
          if (s[i].host) cudaFreeHost(s[i].host);
          if (s[i].segs_h) cudaFreeHost(s[i].segs_h);
          if (s[i].dev) cudaFree(s[i].dev);
          if (s[i].segs_d) cudaFree(s[i].segs_d);
        }
      }
    } freer{slot};
    for (auto& sl : slot) {
      sl.seg_cap = kChunk / (4 + 8 + row_bytes) + 1;
      HMI_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&sl.host), kChunk, cudaHostAllocDefault));
      HMI_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&sl.segs_h), sl.seg_cap * sizeof(int4), cudaHostAllocDefault));
      HMI_CUDA(cudaMalloc(reinterpret_cast<void**>(&sl.dev), kChunk));
      HMI_CUDA(cudaMalloc(reinterpret_cast<void**>(&sl.segs_d), sl.seg_cap * sizeof(int4)));
      HMI_CUDA(cudaEventCreateWithFlags(&sl.done, cudaEventDisableTiming));
    }
    const double t_alloc = now() - t_a;
    std::vector<uint32_t> key_len;
    std::vector<uint32_t> keys;
    key_len.reserve(count);
    keys.reserve(static_cast<size_t>(count) * ngram);
    uint64_t row = 0;       // rows streamed so far (relative to rep_rows)
    uint32_t entries = 0;
    size_t carry = 0;       // bytes of a partial entry carried to the next chunk
    uint64_t chunk_at = off; // file offset of the current chunk's first byte
    int k = 0;
    const uint8_t* prev = nullptr;
    while (entries < count) {
      Slot& sl = slot[k];
      double t0 = now();
      HMI_CUDA(cudaEventSynchronize(sl.done));  // the GPU is done with this slot's last chunk
      t_wait += now() - t0;
      t0 = now();
      if (carry) std::memmove(sl.host, prev, carry);
      const size_t want = std::min<uint64_t>(kChunk - carry, file_size - (chunk_at + carry));
      // page-cache copies are bound by one core's memcpy: read the chunk's quarters in parallel
      const size_t got = read_parallel(fileno(f), sl.host + carry, want, chunk_at + carry);
      if (got != want) fail("read failed", chunk_at + carry);
      t_read += now() - t0;
      t0 = now();
      const size_t avail = carry + got;
      if (avail == 0) fail("unexpected end of file", chunk_at);
      size_t p = 0;
      size_t nseg = 0;
      while (entries < count) {
        if (p + 4 > avail) break;
        uint32_t kl;
        std::memcpy(&kl, sl.host + p, 4);
        if (kl == 0 || kl > ngram)
          fail("entry key length " + std::to_string(kl) + " outside [1, " + std::to_string(ngram) + "]", chunk_at + p);
        const size_t need = 4 + 4 * size_t(kl) + 8 + kl * row_bytes;
        if (p + need > avail) break;
        uint64_t fr;
        std::memcpy(&fr, sl.host + p + 4 + 4 * kl, 8);
        if (fr == 0) fail("entry frequency must be >= 1", chunk_at + p);
        key_len.push_back(kl);
        const uint32_t* kp = reinterpret_cast<const uint32_t*>(sl.host + p + 4);
        for (uint32_t j = 0; j < ngram; ++j) keys.push_back(j < kl ? kp[j] : 0);
        sl.segs_h[nseg++] = make_int4(static_cast<int>(p + 4 + 4 * kl + 8),
                                      static_cast<int>(row & 0x7fffffff), static_cast<int>(row >> 31),
                                      static_cast<int>(kl));
        row += kl;
        ++entries;
        p += need;
      }
      if (p == 0 && entries < count) {
        if (avail < kChunk && chunk_at + avail >= file_size) fail("unexpected end of file", chunk_at + avail);
        fail("PLT1 entry larger than the ingest chunk", chunk_at);
      }
      t_parse += now() - t0;
      if (nseg) {
        HMI_CUDA(cudaMemcpyAsync(sl.dev, sl.host, p, cudaMemcpyHostToDevice, c.copy));
        HMI_CUDA(cudaMemcpyAsync(sl.segs_d, sl.segs_h, nseg * sizeof(int4), cudaMemcpyHostToDevice, c.copy));
        launch_scatter_rows(sl.dev, sl.segs_d, static_cast<int>(nseg), dst_base, static_cast<int>(d), c.copy);
        HMI_CUDA(cudaEventRecord(sl.done, c.copy));
      }
      carry = avail - p;
      prev = sl.host + p;
      chunk_at += p;
      k ^= 1;
    }
    if (chunk_at != file_size) fail("trailing bytes after payload", chunk_at);
    check_new_version(c, version, parent);
    double t0 = now();
    HMI_CUDA(cudaStreamSynchronize(c.copy));
    t_wait += now() - t0;
    t0 = now();
    // keys into the hash; duplicates / vocabulary as hmi_gpu_upload_table (the rows streamed
    // above are only reachable once the hash is committed)
    uint64_t rows = 0;
    auto staged = stage_keys(c, version, count, key_len.data(), keys.data(), &rows);
    HMI_CHECK(rows == row, HMI_SCHEDULING_BUG, "streamed row count mismatch");
    commit_version(c, version, parent, count, rows, staged);
    if (dbg)
      std::fprintf(stderr, "[ingest] alloc+reserve %.1f ms, read %.1f, parse %.1f, gpu wait %.1f, hash+commit %.1f, total %.1f\n",
                   t_alloc, t_read, t_parse, t_wait, now() - t0, now() - t_a);
    if (version_out) *version_out = version;
    if (parent_out) *parent_out = parent;
  });
}

int hmi_gpu_register_task(hmi_gpu_ctx* ctx, uint32_t task_idx, const float* adapter_f32) {
  using namespace hmi_b200;
  return guarded([&] {
    Ctx& c = ctx->impl;
    std::lock_guard<std::mutex> lock(c.mu);
    HMI_CHECK(task_idx < c.store.size(), HMI_CONFIG_ERROR, "task index exceeds max_tasks");
    if (c.store[task_idx]) throw HmiError(HMI_CONFLICT_ERROR, "adapter set for task already registered");
    uint8_t* p = c.store_alloc();
    try {
      c.convert_adapter(adapter_f32, p);
      c.fold_adapters(&p, 1);
    } catch (...) {
      c.free_blocks.push_back(p);
      throw;
    }
    c.store[task_idx] = p;
    c.pool->set_task(task_idx, static_cast<uint32_t>(c.L), c.ref_layer_bytes);
  });
}

// Bulk registration (10k-tenant start-up): indices validated up front,
// host blocks taken under the lock, then the adapters are read / converted on `threads` host
// threads; all-or-nothing (the first failing task, in index order, is reported).
static int register_many(hmi_gpu_ctx* ctx, uint32_t n, const uint32_t* task_idx, uint32_t threads,
                         const std::function<void(uint32_t, std::vector<float>&, uint8_t*)>& fill) {
  using namespace hmi_b200;
  return guarded([&] {
    HMI_CHECK(ctx != nullptr && (n == 0 || task_idx != nullptr), HMI_CONFIG_ERROR, "null argument");
    Ctx& c = ctx->impl;
    std::lock_guard<std::mutex> lock(c.mu);
    std::set<uint32_t> seen;
    for (uint32_t k = 0; k < n; ++k) {
      HMI_CHECK(task_idx[k] < c.store.size(), HMI_CONFIG_ERROR, "task index exceeds max_tasks");
      if (c.store[task_idx[k]] || !seen.insert(task_idx[k]).second)
        throw HmiError(HMI_CONFLICT_ERROR, "adapter set for task already registered");
    }
    std::vector<uint8_t*> blocks(n);
    for (uint32_t k = 0; k < n; ++k) blocks[k] = c.store_alloc();
    const uint32_t hw = std::max(1u, std::thread::hardware_concurrency());
    const uint32_t nt = std::min<uint32_t>(std::max<uint32_t>(1, n), threads ? threads : std::min(hw, 32u));
    std::atomic<uint32_t> next{0};
    std::vector<int> code(n, HMI_OK);
    std::vector<std::string> msg(n);
    auto work = [&] {
      std::vector<float> scratch;
      for (uint32_t k; (k = next.fetch_add(1)) < n;) {
        try {
          fill(k, scratch, blocks[k]);
        } catch (const HmiError& e) {
          code[k] = e.code;
          msg[k] = e.what();
        } catch (const std::exception& e) {
          code[k] = HMI_CAPACITY_ERROR;
          msg[k] = e.what();
        }
      }
    };
    std::vector<std::thread> pool;
    for (uint32_t t = 1; t < nt; ++t) pool.emplace_back(work);
    work();
    for (auto& t : pool) t.join();
    for (uint32_t k = 0; k < n; ++k) {
      if (code[k] != HMI_OK) {
        for (uint8_t* b : blocks) c.free_blocks.push_back(b);
        throw HmiError(code[k], "task " + std::to_string(task_idx[k]) + ": " + msg[k]);
      }
    }
    try {
      c.fold_adapters(blocks.data(), blocks.size());
    } catch (...) {
      for (uint8_t* b : blocks) c.free_blocks.push_back(b);
      throw;
    }
    for (uint32_t k = 0; k < n; ++k) {
      c.store[task_idx[k]] = blocks[k];
      c.pool->set_task(task_idx[k], static_cast<uint32_t>(c.L), c.ref_layer_bytes);
    }
  });
}

int hmi_gpu_register_tasks(hmi_gpu_ctx* ctx, uint32_t n, const uint32_t* task_idx,
                           const float* const* adapter_f32, uint32_t threads) {
  using namespace hmi_b200;
  if (n && !adapter_f32) {
    set_last_error("null argument");
    return HMI_CONFIG_ERROR;
  }
  return register_many(ctx, n, task_idx, threads, [&](uint32_t k, std::vector<float>&, uint8_t* blk) {
    HMI_CHECK(adapter_f32[k] != nullptr, HMI_CONFIG_ERROR, "null adapter");
    ctx->impl.convert_adapter(adapter_f32[k], blk);
  });
}

int hmi_gpu_register_task_files(hmi_gpu_ctx* ctx, uint32_t n, const uint32_t* task_idx,
                                const char* const* adp1_paths, uint32_t threads) {
  using namespace hmi_b200;
  if (n && !adp1_paths) {
    set_last_error("null argument");
    return HMI_CONFIG_ERROR;
  }
  return register_many(ctx, n, task_idx, threads, [&](uint32_t k, std::vector<float>& body, uint8_t* blk) {
    const Ctx& c = ctx->impl;
    body.resize((static_cast<size_t>(c.d) * c.r * 2 + c.r + c.d) * c.L);
    load_adp1_expect(adp1_paths[k], static_cast<uint32_t>(c.L), static_cast<uint32_t>(c.d),
                     static_cast<uint32_t>(c.r), body.data());
    c.convert_adapter(body.data(), blk);
  });
}

static void evict_task_slots(Ctx& c, uint32_t task, bool remove) {
  using namespace hmi_b200;
  std::vector<PoolFree> freed;
  if (remove) {
    c.pool->remove_task(task, &freed);
  } else {
    c.pool->evict(task, &freed);
  }
  // the freed entries are all of one task's row: one write of L entries
  if (!freed.empty()) {
    std::vector<int32_t> row(c.L);
    for (int l = 0; l < c.L; ++l) row[l] = remove ? -1 : c.pool->slot_of(task, static_cast<uint32_t>(l));
    for (const PoolFree& fr : freed) row[fr.layer] = -1;
    HMI_CUDA(cudaMemcpy(c.d_slot_of.p + static_cast<size_t>(task) * c.L, row.data(), 4 * c.L,
                        cudaMemcpyHostToDevice));
  }
}

int hmi_gpu_replace_task(hmi_gpu_ctx* ctx, uint32_t task_idx, const float* adapter_f32) {
  using namespace hmi_b200;
  return guarded([&] {
    Ctx& c = ctx->impl;
    std::lock_guard<std::mutex> lock(c.mu);
    HMI_CUDA(cudaSetDevice(c.device));
    c.reap(true);
    if (task_idx >= c.store.size() || !c.store[task_idx])
      throw HmiError(HMI_ROUTING_ERROR, "no adapter set registered for task");
    HMI_CHECK(!c.exported.count(task_idx), HMI_CONFLICT_ERROR, "task is exported to a peer engine");
    c.convert_adapter(adapter_f32, c.store[task_idx]);
    c.fold_adapters(&c.store[task_idx], 1);
    evict_task_slots(c, task_idx, false);
  });
}

int hmi_gpu_unregister_task(hmi_gpu_ctx* ctx, uint32_t task_idx) {
  using namespace hmi_b200;
  return guarded([&] {
    Ctx& c = ctx->impl;
    std::lock_guard<std::mutex> lock(c.mu);
    HMI_CUDA(cudaSetDevice(c.device));
    c.reap(true);
    if (task_idx >= c.store.size() || !c.store[task_idx]) return;  // AdapterStore::erase is a no-op
    HMI_CHECK(!c.exported.count(task_idx), HMI_CONFLICT_ERROR, "task is exported to a peer engine");
    evict_task_slots(c, task_idx, true);
    c.free_blocks.push_back(c.store[task_idx]);
    c.store[task_idx] = nullptr;
  });
}

// ---- peer rebalancing ---------------------------------------------
// Out-of-band residency change (nothing in flight): the slot-table entries of the records'
// evictions and loads are written directly; the batch path ships the same entries as deltas.
static void write_slot_entries(hmi_b200::Ctx& c, const std::vector<hmi_b200::PoolRecord>& recs) {
  using namespace hmi_b200;
  std::set<uint32_t> touched;
  for (const PoolRecord& rec : recs) {
    for (const PoolFree& fr : rec.freed) touched.insert(fr.task);
    if (!rec.loads.empty()) touched.insert(rec.task);
  }
  // one row of L entries per touched task (rows are contiguous in the slot table)
  std::vector<int32_t> row(c.L);
  for (uint32_t t : touched) {
    for (int l = 0; l < c.L; ++l) row[l] = c.pool->slot_of(t, static_cast<uint32_t>(l));
    HMI_CUDA(cudaMemcpy(c.d_slot_of.p + size_t(t) * c.L, row.data(), 4 * c.L, cudaMemcpyHostToDevice));
  }
}

int hmi_gpu_export_task(hmi_gpu_ctx* src, uint32_t task_idx, hmi_task_export* out) {
  using namespace hmi_b200;
  return guarded([&] {
    HMI_CHECK(src != nullptr && out != nullptr, HMI_CONFIG_ERROR, "null argument");
    Ctx& c = src->impl;
    std::lock_guard<std::mutex> lock(c.mu);
    HMI_CUDA(cudaSetDevice(c.device));
    HMI_CHECK(c.L <= HMI_EXPORT_MAX_LAYERS, HMI_CONFIG_ERROR, "too many higher layers to export");
    if (task_idx >= c.store.size() || !c.store[task_idx])
      throw HmiError(HMI_ROUTING_ERROR, "no adapter set registered for task");
    c.reap(true);
    // every layer resident under the LRU law; missing layers come from the pinned host copy
    auto recs = c.pool->ensure_resident({task_idx});
    for (const PoolRecord& rec : recs) {
      for (const PoolLoad& ld : rec.loads) {
        HMI_CUDA(cudaMemcpyAsync(c.arena.p + size_t(ld.slot) * c.slot_bytes,
                                 c.store[rec.task] + size_t(ld.layer) * c.slot_bytes, c.slot_bytes,
                                 cudaMemcpyHostToDevice, c.copy));
        c.bytes_copied += c.slot_bytes;
        ++c.n_copies;
      }
    }
    HMI_CUDA(cudaStreamSynchronize(c.copy));
    write_slot_entries(c, recs);
    c.pool->pin({task_idx});
    ++c.exported[task_idx];
    std::memset(out, 0, sizeof(*out));
    out->device = c.device;
    out->pid = static_cast<int32_t>(getpid());
    out->arena = reinterpret_cast<uint64_t>(c.arena.p);
    if (c.ipc_state == 0) {
      c.ipc_state = cudaIpcGetMemHandle(&c.ipc_handle, c.arena.p) == cudaSuccess ? 1 : -1;
      (void)cudaGetLastError();  // not exportable: same-process peers still use the raw address
    }
    static_assert(sizeof(c.ipc_handle) == sizeof(out->ipc_handle), "IPC handle size");
    if (c.ipc_state == 1) std::memcpy(out->ipc_handle, &c.ipc_handle, sizeof(c.ipc_handle));
    out->slot_bytes = c.slot_bytes;
    out->fingerprint = c.fingerprint();
    out->layers = static_cast<uint32_t>(c.L);
    out->task_idx = task_idx;
    for (int l = 0; l < c.L; ++l) out->slot[l] = c.pool->slot_of(task_idx, static_cast<uint32_t>(l));
  });
}

int hmi_gpu_import_task(hmi_gpu_ctx* dst, uint32_t task_idx, const hmi_task_export* ex,
                        const float* adapter_f32, uint64_t* peer_bytes) {
  using namespace hmi_b200;
  return guarded([&] {
    HMI_CHECK(dst != nullptr && ex != nullptr, HMI_CONFIG_ERROR, "null argument");
    Ctx& c = dst->impl;
    std::lock_guard<std::mutex> lock(c.mu);
    HMI_CUDA(cudaSetDevice(c.device));
    HMI_CHECK(task_idx < c.store.size(), HMI_CONFIG_ERROR, "task index exceeds max_tasks");
    if (c.store[task_idx]) throw HmiError(HMI_CONFLICT_ERROR, "adapter set for task already registered");
    HMI_CHECK(ex->fingerprint == c.fingerprint() && ex->layers == static_cast<uint32_t>(c.L) &&
                  ex->slot_bytes == c.slot_bytes,
              HMI_CONFIG_ERROR,
              "exported adapter set does not match this engine's model / bottleneck / precision");
    for (int l = 0; l < c.L; ++l)
      HMI_CHECK(ex->slot[l] >= 0, HMI_CONFIG_ERROR, "export holds a non-resident layer");
    const bool local = ex->pid == static_cast<int32_t>(getpid());
    const uint8_t* base = nullptr;
    if (local) {
      base = reinterpret_cast<const uint8_t*>(ex->arena);
      if (ex->device != c.device) {
        int can = 0;
        HMI_CUDA(cudaDeviceCanAccessPeer(&can, c.device, ex->device));
        if (can) {
          const cudaError_t e = cudaDeviceEnablePeerAccess(ex->device, 0);
          if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) HMI_CUDA(e);
          (void)cudaGetLastError();
        }
      }
    } else {
      const std::string key(reinterpret_cast<const char*>(ex->ipc_handle), sizeof(ex->ipc_handle));
      auto it = c.ipc_open.find(key);
      if (it == c.ipc_open.end()) {
        cudaIpcMemHandle_t h;
        std::memcpy(&h, ex->ipc_handle, sizeof(h));
        void* p = nullptr;
        HMI_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
        it = c.ipc_open.emplace(key, p).first;
      }
      base = static_cast<const uint8_t*>(it->second);
    }
    c.reap(true);
    uint8_t* p = c.store_alloc();
    c.store[task_idx] = p;
    c.pool->set_task(task_idx, static_cast<uint32_t>(c.L), c.ref_layer_bytes);
    try {
      auto recs = c.pool->ensure_resident({task_idx});
      uint64_t moved = 0;
      for (const PoolRecord& rec : recs) {
        for (const PoolLoad& ld : rec.loads) {
          uint8_t* to = c.arena.p + size_t(ld.slot) * c.slot_bytes;
          const uint8_t* from = base + size_t(ex->slot[ld.layer]) * c.slot_bytes;
          if (local) {
            HMI_CUDA(cudaMemcpyPeerAsync(to, c.device, from, ex->device, c.slot_bytes, c.copy));
          } else {
            HMI_CUDA(cudaMemcpyAsync(to, from, c.slot_bytes, cudaMemcpyDefault, c.copy));
          }
          moved += c.slot_bytes;
        }
      }
      HMI_CUDA(cudaStreamSynchronize(c.copy));
      write_slot_entries(c, recs);
      if (adapter_f32) {
        c.convert_adapter(adapter_f32, p);
        c.fold_adapters(&p, 1);
      } else {
        // the host copy (for later refills after eviction) is the slot image itself
        for (int l = 0; l < c.L; ++l)
          HMI_CUDA(cudaMemcpyAsync(p + size_t(l) * c.slot_bytes,
                                   c.arena.p + size_t(c.pool->slot_of(task_idx, l)) * c.slot_bytes,
                                   c.slot_bytes, cudaMemcpyDeviceToHost, c.copy));
        HMI_CUDA(cudaStreamSynchronize(c.copy));
      }
      c.peer_bytes += moved;
      if (peer_bytes) *peer_bytes = moved;
    } catch (...) {
      std::vector<PoolFree> freed;
      c.pool->remove_task(task_idx, &freed);
      for (const PoolFree& fr : freed) {
        const int32_t minus1 = -1;
        cudaMemcpy(c.d_slot_of.p + size_t(fr.task) * c.L + fr.layer, &minus1, 4, cudaMemcpyHostToDevice);
      }
      c.free_blocks.push_back(p);
      c.store[task_idx] = nullptr;
      throw;
    }
  });
}

int hmi_gpu_release_export(hmi_gpu_ctx* src, uint32_t task_idx, int drop) {
  using namespace hmi_b200;
  return guarded([&] {
    HMI_CHECK(src != nullptr, HMI_CONFIG_ERROR, "null context");
    Ctx& c = src->impl;
    std::lock_guard<std::mutex> lock(c.mu);
    HMI_CUDA(cudaSetDevice(c.device));
    auto it = c.exported.find(task_idx);
    if (it == c.exported.end()) throw HmiError(HMI_ROUTING_ERROR, "task is not exported");
    c.pool->unpin({task_idx});
    if (--it->second == 0) c.exported.erase(it);
    if (drop) {
      HMI_CHECK(!c.exported.count(task_idx), HMI_CONFLICT_ERROR,
                "task is still exported to another peer engine");
      c.reap(true);
      evict_task_slots(c, task_idx, true);
      c.free_blocks.push_back(c.store[task_idx]);
      c.store[task_idx] = nullptr;
    }
  });
}

int hmi_gpu_register_head(hmi_gpu_ctx* ctx, uint32_t head_idx, uint32_t kind, uint32_t labels,
                          const float* w, const float* b) {
  using namespace hmi_b200;
  return guarded([&] {
    Ctx& c = ctx->impl;
    std::lock_guard<std::mutex> lock(c.mu);
    HMI_CUDA(cudaSetDevice(c.device));
    c.reap(true);
    HMI_CHECK(head_idx < c.h_head_off.size(), HMI_CONFIG_ERROR, "head index exceeds max_heads");
    HMI_CHECK(kind <= 2, HMI_CONFIG_ERROR, "head kind must be 0, 1 or 2");
    HMI_CHECK(labels >= 1, HMI_CONFIG_ERROR, "output head needs at least one label");
    const bool wide = kind == 2 && labels > c.opt.max_labels;  // vocabulary-wide lm head
    HMI_CHECK(labels <= c.opt.max_labels || wide, HMI_CONFIG_ERROR, "head labels exceed max_labels");
    if (c.h_head_kind[head_idx] >= 0) throw HmiError(HMI_CONFLICT_ERROR, "head already registered");
    const size_t n = static_cast<size_t>(c.d) * labels + labels;
    if (c.head_floats + n > c.d_head_arena.n) {
      c.drop_decode_graphs();  // graphs read the head arena by address
      DevBuf<float> grown;
      grown.alloc(std::max(c.head_floats + n, c.d_head_arena.n * 3 / 2 + 1024));
      if (c.head_floats)
        HMI_CUDA(cudaMemcpy(grown.p, c.d_head_arena.p, c.head_floats * 4, cudaMemcpyDeviceToDevice));
      c.d_head_arena.free();
      c.d_head_arena = grown;
      grown.p = nullptr;
    }
    HMI_CUDA(cudaMemcpy(c.d_head_arena.p + c.head_floats, w, static_cast<size_t>(c.d) * labels * 4,
                        cudaMemcpyHostToDevice));
    HMI_CUDA(cudaMemcpy(c.d_head_arena.p + c.head_floats + static_cast<size_t>(c.d) * labels, b,
                        labels * 4, cudaMemcpyHostToDevice));
    c.h_head_off[head_idx] = static_cast<int64_t>(c.head_floats);
    c.h_head_labels[head_idx] = static_cast<int32_t>(labels);
    c.h_head_kind[head_idx] = static_cast<int32_t>(kind);
    c.head_floats += n;
    HMI_CUDA(cudaMemcpy(c.d_head_off.p + head_idx, &c.h_head_off[head_idx], 8, cudaMemcpyHostToDevice));
    HMI_CUDA(cudaMemcpy(c.d_head_labels.p + head_idx, &c.h_head_labels[head_idx], 4, cudaMemcpyHostToDevice));
    HMI_CUDA(cudaMemcpy(c.d_head_kind.p + head_idx, &c.h_head_kind[head_idx], 4, cudaMemcpyHostToDevice));
    if (wide) {
      // 16-bit K-major copy [V_pad][d] for the tcgen05 logits GEMM; padded columns are zero
      Ctx::LmHead h;
      h.V = static_cast<int>(labels);
      h.V_pad = static_cast<int>((labels + 255) / 256 * 256);
      const size_t dd = static_cast<size_t>(c.d);
      std::vector<uint16_t> wt(static_cast<size_t>(h.V_pad) * dd, 0);
      std::vector<float> wtf(static_cast<size_t>(labels) * dd);
      for (size_t i = 0; i < dd; ++i)
        for (size_t j = 0; j < labels; ++j) {
          wt[j * dd + i] = f2h(w[i * labels + j], static_cast<int>(c.opt.precision));
          wtf[j * dd + i] = w[i * labels + j];
        }
      // f32 transpose for the candidates' f64 rescoring: a column of the reference layout is
      // one contiguous row here (coalesced, instead of d scattered 4-byte reads V apart)
      HMI_CUDA(cudaMalloc(&h.wT, wtf.size() * 4));
      HMI_CUDA(cudaMemcpy(h.wT, wtf.data(), wtf.size() * 4, cudaMemcpyHostToDevice));
      std::vector<float> bp(h.V_pad, 0.f);
      std::memcpy(bp.data(), b, labels * 4);
      HMI_CUDA(cudaMalloc(&h.w16, wt.size() * 2));
      HMI_CUDA(cudaMalloc(&h.bias, bp.size() * 4));
      HMI_CUDA(cudaMemcpy(h.w16, wt.data(), wt.size() * 2, cudaMemcpyHostToDevice));
      HMI_CUDA(cudaMemcpy(h.bias, bp.data(), bp.size() * 4, cudaMemcpyHostToDevice));
      const size_t need = static_cast<size_t>(c.Bp) * h.V_pad;
      if (c.lm_logits.n < need) {
        c.drop_decode_graphs();  // graphs write the logits buffer by address
        c.lm_logits.alloc(need);
        for (auto& [id, o] : c.lm_heads) c.build_lm_plan(o);  // logits buffer moved
      }
      c.build_lm_plan(h);
      c.lm_heads[static_cast<int>(head_idx)] = h;
    }
  });
}

int hmi_gpu_bind_instance(hmi_gpu_ctx* ctx, uint32_t instance_idx, uint32_t version_id,
                          uint32_t task_idx, uint32_t head_idx) {
  using namespace hmi_b200;
  return guarded([&] {
    Ctx& c = ctx->impl;
    std::lock_guard<std::mutex> lock(c.mu);
    HMI_CUDA(cudaSetDevice(c.device));
    c.reap(true);
    HMI_CHECK(instance_idx < c.h_inst_task.size(), HMI_CONFIG_ERROR, "instance index exceeds max_instances");
    if (c.h_inst_task[instance_idx] >= 0) throw HmiError(HMI_CONFLICT_ERROR, "instance already bound");
    if (version_id >= c.h_parent.size() || c.h_parent[version_id] == -2)
      throw HmiError(HMI_ROUTING_ERROR, "version " + std::to_string(version_id) + " does not exist");
    if (task_idx >= c.store.size() || !c.store[task_idx])
      throw HmiError(HMI_ROUTING_ERROR, "no adapter set registered for task");
    if (head_idx >= c.h_head_kind.size() || c.h_head_kind[head_idx] < 0)
      throw HmiError(HMI_ROUTING_ERROR, "no output head registered");
    c.h_inst_version[instance_idx] = static_cast<int32_t>(version_id);
    c.h_inst_task[instance_idx] = static_cast<int32_t>(task_idx);
    c.h_inst_head[instance_idx] = static_cast<int32_t>(head_idx);
    HMI_CUDA(cudaMemcpy(c.d_inst_version.p + instance_idx, &c.h_inst_version[instance_idx], 4, cudaMemcpyHostToDevice));
    HMI_CUDA(cudaMemcpy(c.d_inst_task.p + instance_idx, &c.h_inst_task[instance_idx], 4, cudaMemcpyHostToDevice));
    HMI_CUDA(cudaMemcpy(c.d_inst_head.p + instance_idx, &c.h_inst_head[instance_idx], 4, cudaMemcpyHostToDevice));
  });
}

int hmi_gpu_unbind_instance(hmi_gpu_ctx* ctx, uint32_t instance_idx) {
  using namespace hmi_b200;
  return guarded([&] {
    Ctx& c = ctx->impl;
    std::lock_guard<std::mutex> lock(c.mu);
    HMI_CUDA(cudaSetDevice(c.device));
    c.reap(true);
    if (instance_idx >= c.h_inst_task.size()) return;
    c.h_inst_version[instance_idx] = c.h_inst_task[instance_idx] = c.h_inst_head[instance_idx] = -1;
    const int32_t m1 = -1;
    HMI_CUDA(cudaMemcpy(c.d_inst_version.p + instance_idx, &m1, 4, cudaMemcpyHostToDevice));
    HMI_CUDA(cudaMemcpy(c.d_inst_task.p + instance_idx, &m1, 4, cudaMemcpyHostToDevice));
    HMI_CUDA(cudaMemcpy(c.d_inst_head.p + instance_idx, &m1, 4, cudaMemcpyHostToDevice));
  });
}

static void fill_trace(const std::vector<hmi_b200::PoolRecord>& recs, const std::vector<int32_t>& layer_tag,
                       hmi_load_record* trace, uint32_t trace_cap, uint32_t* evicted,
                       uint32_t evicted_cap, uint32_t* n_trace) {
  uint32_t ev = 0;
  for (size_t i = 0; i < recs.size() && i < trace_cap; ++i) {
    hmi_load_record& t = trace[i];
    t.task = recs[i].task;
    t.layer = layer_tag[i];
    t.hit = recs[i].hit ? 1 : 0;
    t.bytes = recs[i].bytes;
    t.n_evicted = static_cast<uint32_t>(recs[i].evicted.size());
    t.evicted_offset = ev;
    t.pad = 0;
    for (uint32_t e : recs[i].evicted) {
      if (evicted && ev < evicted_cap) evicted[ev] = e;
      ++ev;
    }
  }
  if (n_trace) *n_trace = static_cast<uint32_t>(recs.size());
}

int hmi_gpu_infer_batch(hmi_gpu_ctx* ctx, uint32_t n_req, const uint32_t* instance_idx,
                        const uint32_t* tokens, uint32_t stride, const uint32_t* lens,
                        float* scores, int32_t* labels, int32_t* tags, hmi_load_record* trace,
                        uint32_t trace_cap, uint32_t* evicted, uint32_t evicted_cap,
                        uint32_t* n_trace) {
  using namespace hmi_b200;
  return guarded([&] {
    Ctx& c = ctx->impl;
    std::lock_guard<std::mutex> lock(c.mu);
    HMI_CUDA(cudaSetDevice(c.device));
    std::vector<PoolRecord> recs;
    std::vector<int32_t> tag;
    const bool want = trace || n_trace;
    const int si = c.submit(n_req, instance_idx, tokens, nullptr, stride, lens, nullptr, 0, nullptr,
                            nullptr, want ? &recs : nullptr, want ? &tag : nullptr);
    Staging& st = c.stg[si];
    HMI_CUDA(cudaEventSynchronize(st.done));
    if (tags) {
      HMI_CUDA(cudaMemcpy(st.tags, c.d_tags.p, static_cast<size_t>(n_req) * c.last_S * 4, cudaMemcpyDeviceToHost));
      for (uint32_t i = 0; i < n_req; ++i) {
        for (uint32_t p = 0; p < stride; ++p)
          tags[static_cast<size_t>(i) * stride + p] = p < lens[i] ? st.tags[static_cast<size_t>(i) * c.last_S + p] : -1;
      }
    }
    const int err = *st.err;
    *st.err = 0;
    std::memcpy(scores, st.scores, static_cast<size_t>(n_req) * c.opt.max_labels * 4);
    std::memcpy(labels, st.labels, n_req * 4);
    if (c.prof) c.prof_collect();
    c.reap(false);
    if (want) fill_trace(recs, tag, trace, trace_cap, evicted, evicted_cap, n_trace);
    if (err) throw HmiError(err, "device-side error in batch (status " + std::to_string(err) + ")");
  });
}

int hmi_gpu_check_adapter_dims(hmi_gpu_ctx* ctx, uint32_t layers, uint32_t d, uint32_t r) {
  using namespace hmi_b200;
  return guarded([&] {
    HMI_CHECK(ctx != nullptr, HMI_CONFIG_ERROR, "null context");
    const Ctx& c = ctx->impl;
    HMI_CHECK(layers == static_cast<uint32_t>(c.L) && d == static_cast<uint32_t>(c.d) &&
                  r == static_cast<uint32_t>(c.r),
              HMI_DIMENSION_ERROR,
              "adapter set (" + std::to_string(layers) + " layers, d " + std::to_string(d) + ", r " +
                  std::to_string(r) + ") does not match the model (" + std::to_string(c.L) +
                  " higher layers, d " + std::to_string(c.d) + ", r " + std::to_string(c.r) + ")");
  });
}

int hmi_gpu_trace(hmi_gpu_ctx* ctx, int enable) {
  using namespace hmi_b200;
  return guarded([&] {
    Ctx& c = ctx->impl;
    std::lock_guard<std::mutex> lock(c.mu);
    HMI_CUDA(cudaSetDevice(c.device));
    HMI_CUDA(cudaDeviceSynchronize());
    for (auto& e : c.trace_evs) {
      if (e.a) cudaEventDestroy(e.a);
      if (e.b) cudaEventDestroy(e.b);
    }
    c.trace_evs.clear();
    if (!c.trace_epoch) HMI_CUDA(cudaEventCreate(&c.trace_epoch));
    c.trace_on = enable != 0;
    if (c.trace_on) {  // device idle: the epoch event and the host origin coincide
      HMI_CUDA(cudaEventRecord(c.trace_epoch, c.compute));
      HMI_CUDA(cudaEventSynchronize(c.trace_epoch));
      c.trace_host0 = std::chrono::steady_clock::now();
    }
  });
}

int hmi_gpu_stage_trace(hmi_gpu_ctx* ctx, hmi_stage_record* out, uint32_t cap, uint32_t* n) {
  using namespace hmi_b200;
  return guarded([&] {
    Ctx& c = ctx->impl;
    std::lock_guard<std::mutex> lock(c.mu);
    HMI_CUDA(cudaSetDevice(c.device));
    HMI_CHECK(c.trace_epoch != nullptr, HMI_CONFIG_ERROR, "tracing was never enabled");
    HMI_CUDA(cudaDeviceSynchronize());
    uint32_t k = 0;
    double prev_end = 0.0;  // compute-stream end of the previous record (head start)
    for (const auto& e : c.trace_evs) {
      hmi_stage_record r{};
      r.batch = e.batch;
      r.stage = static_cast<uint32_t>(e.stage);
      r.layer = e.layer;
      r.worker = static_cast<uint32_t>(e.worker);
      if (e.worker == kWorkerCpu) {
        r.start_ms = e.host_a;
        r.end_ms = e.host_b;
      } else {
        float ms = 0.f;
        HMI_CUDA(cudaEventElapsedTime(&ms, c.trace_epoch, e.a));
        r.start_ms = ms;
        if (e.b) {
          HMI_CUDA(cudaEventElapsedTime(&ms, c.trace_epoch, e.b));
          r.end_ms = ms;
        } else {  // head: from the end of the batch's last layer to this mark
          r.end_ms = r.start_ms;
          r.start_ms = prev_end;
        }
        if (e.worker == kWorkerCompute) prev_end = r.end_ms;
      }
      if (k < cap && out) out[k] = r;
      ++k;
    }
    if (n) *n = k;
  });
}

int hmi_gpu_submit_batch(hmi_gpu_ctx* ctx, uint32_t n_req, const uint32_t* instance_idx,
                         const uint32_t* tokens, uint32_t stride, const uint32_t* lens,
                         uint64_t* ticket) {
  using namespace hmi_b200;
  return guarded([&] {
    HMI_CHECK(ticket != nullptr, HMI_CONFIG_ERROR, "null ticket");
    Ctx& c = ctx->impl;
    std::lock_guard<std::mutex> lock(c.mu);
    HMI_CUDA(cudaSetDevice(c.device));
    const int si = c.submit(n_req, instance_idx, tokens, nullptr, stride, lens, nullptr, 0, nullptr,
                            nullptr, nullptr, nullptr);
    Staging& st = c.stg[si];
    st.held = true;
    st.ticket = ++c.next_ticket;
    st.n_req = n_req;
    *ticket = st.ticket;
  });
}

int hmi_gpu_wait_batch(hmi_gpu_ctx* ctx, uint64_t ticket, float* scores, int32_t* labels) {
  using namespace hmi_b200;
  return guarded([&] {
    Ctx& c = ctx->impl;
    std::lock_guard<std::mutex> lock(c.mu);
    HMI_CUDA(cudaSetDevice(c.device));
    Staging* st = nullptr;
    for (Staging& x : c.stg)
      if (x.held && x.ticket == ticket) st = &x;
    HMI_CHECK(st != nullptr, HMI_CONFIG_ERROR, "unknown or already collected ticket");
    HMI_CUDA(cudaEventSynchronize(st->done));
    st->held = false;
    const int err = *st->err;
    *st->err = 0;
    if (scores) std::memcpy(scores, st->scores, static_cast<size_t>(st->n_req) * c.opt.max_labels * 4);
    if (labels) std::memcpy(labels, st->labels, st->n_req * 4);
    if (c.prof) c.prof_collect();
    c.reap(false);
    if (err) throw HmiError(err, "device-side error in batch (status " + std::to_string(err) + ")");
  });
}

int hmi_gpu_generate(hmi_gpu_ctx* ctx, uint32_t n_req, const uint32_t* instance_idx,
                     const uint32_t* tokens, uint32_t stride, const uint32_t* lens,
                     uint32_t n_new, int32_t* out_tokens, float* out_logits) {
  using namespace hmi_b200;
  return guarded([&] {
    Ctx& c = ctx->impl;
    std::lock_guard<std::mutex> lock(c.mu);
    HMI_CUDA(cudaSetDevice(c.device));
    HMI_CHECK(n_new >= 1 && out_tokens, HMI_CONFIG_ERROR, "generate: n_new >= 1 and out_tokens required");
    const int si = c.submit(n_req, instance_idx, tokens, nullptr, stride, lens, nullptr, 0, nullptr,
                            nullptr, nullptr, nullptr, n_new);
    Staging& st = c.stg[si];
    HMI_CUDA(cudaEventSynchronize(st.done));
    const size_t T = c.opt.max_new_tokens;
    HMI_CUDA(cudaMemcpy2D(out_tokens, n_new * 4, c.gen_out.p, T * 4, n_new * 4, n_req,
                          cudaMemcpyDeviceToHost));
    if (out_logits) {
      HMI_CUDA(cudaMemcpy2D(out_logits, n_new * 4, c.gen_logit.p, T * 4, n_new * 4, n_req,
                            cudaMemcpyDeviceToHost));
    }
    const int err = *st.err;
    *st.err = 0;
    if (c.prof) c.prof_collect();
    c.reap(false);
    if (err) throw HmiError(err, "device-side error in batch (status " + std::to_string(err) + ")");
  });
}

int hmi_gpu_infer_batch_device(hmi_gpu_ctx* ctx, uint32_t n_req, const uint32_t* instance_idx,
                               const uint32_t* d_tokens, uint32_t stride,
                               const uint32_t* d_lens, uint32_t max_len, float* d_scores,
                               int32_t* d_labels) {
  using namespace hmi_b200;
  return guarded([&] {
    Ctx& c = ctx->impl;
    std::lock_guard<std::mutex> lock(c.mu);
    HMI_CUDA(cudaSetDevice(c.device));
    c.reap(false);
    c.raise_sticky();
    c.submit(n_req, instance_idx, nullptr, d_tokens, stride, nullptr, d_lens, max_len, d_scores,
             d_labels, nullptr, nullptr);
  });
}

int hmi_gpu_synchronize(hmi_gpu_ctx* ctx) {
  using namespace hmi_b200;
  return guarded([&] {
    Ctx& c = ctx->impl;
    std::lock_guard<std::mutex> lock(c.mu);
    HMI_CUDA(cudaSetDevice(c.device));
    c.reap(true);  // latches the first device-side error of the retired batches
    HMI_CUDA(cudaStreamSynchronize(c.compute));
    if (c.prof) c.prof_collect();
    c.raise_sticky();
  });
}

void* hmi_gpu_stream(hmi_gpu_ctx* ctx) { return ctx ? static_cast<void*>(ctx->impl.compute) : nullptr; }

int hmi_gpu_debug_routing(hmi_gpu_ctx* ctx, int32_t* version, int32_t* task, int32_t* head,
                          int32_t* slots) {
  using namespace hmi_b200;
  return guarded([&] {
    Ctx& c = ctx->impl;
    std::lock_guard<std::mutex> lock(c.mu);
    HMI_CUDA(cudaSetDevice(c.device));
    HMI_CUDA(cudaStreamSynchronize(c.compute));
    const uint32_t n = c.last_n;
    if (version) HMI_CUDA(cudaMemcpy(version, c.d_req_version.p, n * 4, cudaMemcpyDeviceToHost));
    if (task) HMI_CUDA(cudaMemcpy(task, c.d_req_task.p, n * 4, cudaMemcpyDeviceToHost));
    if (head) HMI_CUDA(cudaMemcpy(head, c.d_req_head.p, n * 4, cudaMemcpyDeviceToHost));
    if (slots) {
      const uint32_t tpr = c.last_S / 128;
      std::vector<int32_t> t(static_cast<size_t>(c.L) * c.tile_stride);
      HMI_CUDA(cudaMemcpy(t.data(), c.d_tile_slot.p, t.size() * 4, cudaMemcpyDeviceToHost));
      for (int l = 0; l < c.L; ++l)
        for (uint32_t i = 0; i < n; ++i) slots[static_cast<size_t>(l) * n + i] = t[static_cast<size_t>(l) * c.tile_stride + i * tpr];
    }
  });
}

int hmi_gpu_debug_gather(hmi_gpu_ctx* ctx, int32_t* rows, int32_t* levels, uint32_t* S) {
  using namespace hmi_b200;
  return guarded([&] {
    Ctx& c = ctx->impl;
    std::lock_guard<std::mutex> lock(c.mu);
    HMI_CUDA(cudaSetDevice(c.device));
    HMI_CUDA(cudaStreamSynchronize(c.compute));
    const size_t n = static_cast<size_t>(c.last_n) * c.last_S * c.ngram;
    if (rows) HMI_CUDA(cudaMemcpy(rows, c.d_gather.p, n * 4, cudaMemcpyDeviceToHost));
    if (levels) HMI_CUDA(cudaMemcpy(levels, c.d_levels.p, n * 4, cudaMemcpyDeviceToHost));
    if (S) *S = c.last_S;
  });
}

int hmi_gpu_set_debug(hmi_gpu_ctx* ctx, uint32_t flags) {
  using namespace hmi_b200;
  return guarded([&] {
    Ctx& c = ctx->impl;
    std::lock_guard<std::mutex> lock(c.mu);
    HMI_CUDA(cudaSetDevice(c.device));
    c.debug_flags = flags;
    if ((flags & 1) && !c.h64.p) c.h64.alloc(static_cast<size_t>(c.max_rows) * c.d);
  });
}

int hmi_gpu_debug_h0(hmi_gpu_ctx* ctx, double* out) {
  using namespace hmi_b200;
  return guarded([&] {
    Ctx& c = ctx->impl;
    std::lock_guard<std::mutex> lock(c.mu);
    HMI_CHECK(c.h64.p, HMI_CONFIG_ERROR, "enable debug flag 1 before the batch");
    HMI_CUDA(cudaStreamSynchronize(c.compute));
    HMI_CUDA(cudaMemcpy(out, c.h64.p, static_cast<size_t>(c.last_n) * c.last_S * c.d * 8, cudaMemcpyDeviceToHost));
  });
}

int hmi_gpu_debug_hidden(hmi_gpu_ctx* ctx, float* out) {
  using namespace hmi_b200;
  return guarded([&] {
    Ctx& c = ctx->impl;
    std::lock_guard<std::mutex> lock(c.mu);
    HMI_CUDA(cudaStreamSynchronize(c.compute));
    HMI_CUDA(cudaMemcpy(out, c.h32.p, static_cast<size_t>(c.last_n) * c.last_S * c.d * 4, cudaMemcpyDeviceToHost));
  });
}

int hmi_gpu_pool_stats(hmi_gpu_ctx* ctx, uint64_t* out) {
  using namespace hmi_b200;
  return guarded([&] {
    Ctx& c = ctx->impl;
    std::lock_guard<std::mutex> lock(c.mu);
    out[0] = c.pool->hits();
    out[1] = c.pool->loads();
    out[2] = c.pool->resident_bytes();
    out[3] = c.pool->max_resident_bytes_seen();
    out[4] = c.pool->resident_task_count();
    out[5] = c.pool->capacity_bytes();
    out[6] = c.pool->physical_slots();
    out[7] = c.bytes_copied;
  });
}

int hmi_gpu_pool_slot(hmi_gpu_ctx* ctx, uint32_t task_idx, uint32_t layer, int32_t* slot) {
  using namespace hmi_b200;
  return guarded([&] {
    Ctx& c = ctx->impl;
    std::lock_guard<std::mutex> lock(c.mu);
    *slot = c.pool->slot_of(task_idx, layer);
  });
}

int hmi_gpu_profile(hmi_gpu_ctx* ctx, int enable) {
  using namespace hmi_b200;
  return guarded([&] {
    Ctx& c = ctx->impl;
    std::lock_guard<std::mutex> lock(c.mu);
    HMI_CUDA(cudaSetDevice(c.device));
    c.prof_collect();
    c.prof = enable != 0;
    for (int i = 0; i < HMI_PROF_CLASSES; ++i) {
      c.prof_ms[i] = 0;
      c.prof_cnt[i] = 0;
    }
  });
}

int hmi_gpu_profile_read(hmi_gpu_ctx* ctx, double* ms, uint64_t* count) {
  using namespace hmi_b200;
  return guarded([&] {
    Ctx& c = ctx->impl;
    std::lock_guard<std::mutex> lock(c.mu);
    HMI_CUDA(cudaSetDevice(c.device));
    c.prof_collect();
    for (int i = 0; i < HMI_PROF_CLASSES; ++i) {
      if (ms) ms[i] = c.prof_ms[i];
      if (count) count[i] = c.prof_cnt[i];
    }
  });
}

const char* hmi_gpu_profile_name(int cls) {
  return cls >= 0 && cls < HMI_PROF_CLASSES ? hmi_b200::kProfNames[cls] : "";
}

// ---- standalone pool ---------------------------------------------------------
struct hmi_pool {
  std::unique_ptr<hmi_b200::SlotPool> p;
};

int hmi_pool_create(uint64_t capacity_bytes, hmi_pool** out) {
  return guarded([&] {
    auto* h = new hmi_pool;
    h->p = std::make_unique<hmi_b200::SlotPool>(capacity_bytes, 0);
    *out = h;
  });
}

int hmi_pool_create_placed(uint64_t capacity_bytes, uint32_t physical_slots, uint32_t block_len,
                           hmi_pool** out) {
  return guarded([&] {
    HMI_CHECK(out != nullptr && physical_slots > 0, HMI_CONFIG_ERROR, "pool: physical slots");
    auto* h = new hmi_pool;
    h->p = std::make_unique<hmi_b200::SlotPool>(capacity_bytes, physical_slots, block_len);
    *out = h;
  });
}

int hmi_pool_slot(hmi_pool* pool, uint32_t task, uint32_t layer, int32_t* slot) {
  return guarded([&] {
    HMI_CHECK(pool != nullptr && slot != nullptr, HMI_CONFIG_ERROR, "null argument");
    *slot = pool->p->slot_of(task, layer);
  });
}

int hmi_pool_destroy(hmi_pool* pool) {
  delete pool;
  return HMI_OK;
}

int hmi_pool_register(hmi_pool* pool, uint32_t task, uint32_t layers, uint64_t layer_bytes) {
  return guarded([&] {
    if (pool->p->has_task(task)) throw HmiError(HMI_CONFLICT_ERROR, "task already registered");
    pool->p->set_task(task, layers, layer_bytes);
  });
}

int hmi_pool_op(hmi_pool* pool, int op, uint32_t n, const uint32_t* tasks, uint32_t layer,
                hmi_load_record* trace, uint32_t trace_cap, uint32_t* evicted,
                uint32_t evicted_cap, int32_t* n_trace) {
  using namespace hmi_b200;
  return guarded([&] {
    std::vector<uint32_t> v(tasks, tasks + n);
    std::vector<PoolRecord> recs;
    if (n_trace) *n_trace = 0;
    switch (op) {
      case 0:
        try {
          recs = pool->p->ensure_resident(v);
        } catch (...) {
          pool->p->take_partial();
          throw;
        }
        break;
      case 1: {
        auto r = pool->p->try_ensure_layer_resident(v, layer);
        pool->p->take_partial();
        if (!r) {
          if (n_trace) *n_trace = -1;
          return;
        }
        recs = std::move(*r);
        break;
      }
      case 2: pool->p->pin(v); return;
      case 3: pool->p->unpin(v); return;
      case 4: pool->p->touch(v); return;
      case 5:
        if (n_trace) *n_trace = pool->p->evict(v.at(0), nullptr) ? 1 : 0;
        return;
      default: throw HmiError(HMI_CONFIG_ERROR, "unknown pool op");
    }
    std::vector<int32_t> tag(recs.size(), op == 1 ? static_cast<int32_t>(layer) : -1);
    uint32_t cnt = 0;
    fill_trace(recs, tag, trace, trace_cap, evicted, evicted_cap, &cnt);
    if (n_trace) *n_trace = static_cast<int32_t>(cnt);
  });
}

int hmi_pool_stats(hmi_pool* pool, uint64_t* out) {
  return guarded([&] {
    out[0] = pool->p->hits();
    out[1] = pool->p->loads();
    out[2] = pool->p->resident_bytes();
    out[3] = pool->p->max_resident_bytes_seen();
    out[4] = pool->p->resident_task_count();
    out[5] = pool->p->capacity_bytes();
  });
}

}  // extern "C"

extern "C" int hmi_gpu_counters(hmi_gpu_ctx* ctx, uint64_t* out) {
  return guarded([&] {
    Ctx& c = ctx->impl;
    std::lock_guard<std::mutex> lock(c.mu);
    out[0] = c.n_launches;
    out[1] = c.n_batches;
    out[2] = c.n_copies;
    out[3] = c.numa_node < 0 ? ~uint64_t(0) : static_cast<uint64_t>(c.numa_node);
  });
}

// Host -> HBM bandwidth from the pinned adapter store's memory (the source adapter misses
// are copied from) into a scratch buffer, on the context's copy stream. Ranks run it at the
// same time after a barrier, so it measures the concurrent per-GPU rate of the box.
extern "C" int hmi_gpu_h2d_probe(hmi_gpu_ctx* ctx, uint64_t bytes, uint32_t reps, double* gbps) {
  using namespace hmi_b200;
  return guarded([&] {
    HMI_CHECK(ctx != nullptr && gbps != nullptr && bytes > 0 && reps > 0, HMI_CONFIG_ERROR,
              "h2d_probe: bad argument");
    Ctx& c = ctx->impl;
    std::lock_guard<std::mutex> lock(c.mu);
    HMI_CUDA(cudaSetDevice(c.device));
    c.reap(true);
    uint8_t* src = host_alloc_local(bytes, c.numa_node);
    void* dst = nullptr;
    cudaEvent_t a = nullptr, b = nullptr;
    struct Cleanup {
      uint8_t* src; size_t n; void** dst; cudaEvent_t* a; cudaEvent_t* b;
      ~Cleanup() {
        if (*a) cudaEventDestroy(*a);
        if (*b) cudaEventDestroy(*b);
        if (*dst) cudaFree(*dst);
        host_free_local(src, n);
      }
    } cleanup{src, bytes, &dst, &a, &b};
    HMI_CUDA(cudaMalloc(&dst, bytes));
    HMI_CUDA(cudaEventCreate(&a));
    HMI_CUDA(cudaEventCreate(&b));
    HMI_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, c.copy));  // warm
    HMI_CUDA(cudaEventRecord(a, c.copy));
    for (uint32_t i = 0; i < reps; ++i)
      HMI_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, c.copy));
    HMI_CUDA(cudaEventRecord(b, c.copy));
    HMI_CUDA(cudaEventSynchronize(b));
    float ms = 0;
    HMI_CUDA(cudaEventElapsedTime(&ms, a, b));
    *gbps = static_cast<double>(bytes) * reps / (ms * 1e-3) / 1e9;
  });
}
