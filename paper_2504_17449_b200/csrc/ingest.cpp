// SPDX-License-Identifier: Apache-2.0
//
// Artefact ingest: the reference's binary containers read straight
// into the f32 layouts the C ABI consumes — no f64 Matrix round trip — and PLT1 written back,
// so GPU-built PLOT tables persist in the reference's own format.
//
//   PLT1 (proj/src/plot/plot_io.cpp:17-72)        PLOT table: header, then per entry
//                                                  key_len, key, freq, f32 rep rows
//   ADP1 (proj/src/adapters/adapter_set.cpp:27-75) adapter set: task id, layers, d, r, then
//                                                  per layer W_down, b_down, W_up, b_up (f32)
//   HMI1 (proj/src/transformer/model_io.cpp:83-115) model: config, embeddings, lower and
//                                                  higher layers (f32, declaration order)
//
// Validation mirrors the reference readers (bad magic, truncation, trailing bytes, zero
// dimensions, key length outside [1, ngram], zero frequency, duplicate keys -> FormatError with
// the byte offset; io/binary.cpp:62-123), little-endian hosts only (binary.cpp:10-11).
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <set>
#include <string>
#include <vector>

#include "plot_builder.hpp"

namespace hmi_b200 {
namespace {

struct Reader {
  std::vector<uint8_t> data;
  size_t off = 0;

  explicit Reader(const char* path) {
    HMI_CHECK(path != nullptr, HMI_CONFIG_ERROR, "null path");
    FILE* f = std::fopen(path, "rb");
    if (!f) throw HmiError(HMI_FORMAT_ERROR, std::string("cannot open ") + path + " (offset 0)");
    std::fseek(f, 0, SEEK_END);
    const long n = std::ftell(f);
    std::fseek(f, 0, SEEK_SET);
    data.resize(n > 0 ? static_cast<size_t>(n) : 0);
    const size_t got = data.empty() ? 0 : std::fread(data.data(), 1, data.size(), f);
    std::fclose(f);
    if (got != data.size()) throw HmiError(HMI_FORMAT_ERROR, std::string("read failed for ") + path);
  }
  [[noreturn]] void fail(const std::string& what, size_t at) const {
    throw HmiError(HMI_FORMAT_ERROR, what + " (offset " + std::to_string(at) + ")");
  }
  void bytes(void* p, size_t n) {
    if (off + n > data.size()) fail("unexpected end of file", off);
    std::memcpy(p, data.data() + off, n);
    off += n;
  }
  void magic(const char* tag) {
    char got[4];
    bytes(got, 4);
    if (std::memcmp(got, tag, 4) != 0) fail(std::string("bad magic, expected ") + std::string(tag, 4), off - 4);
  }
  uint32_t u32() {
    uint32_t v;
    bytes(&v, 4);
    return v;
  }
  uint64_t u64() {
    uint64_t v;
    bytes(&v, 8);
    return v;
  }
  void f32s(float* out, size_t n) {
    if (off + n * 4 > data.size()) fail("unexpected end of file", off);
    if (out) std::memcpy(out, data.data() + off, n * 4);
    off += n * 4;
  }
  std::string str(size_t max_len = 1u << 20) {
    const size_t at = off;
    const uint32_t len = u32();
    if (len > max_len) fail("string length " + std::to_string(len) + " implausible", at);
    std::string s(len, '\0');
    if (len) bytes(&s[0], len);
    return s;
  }
  void expect_end() const {
    if (off != data.size()) fail("trailing bytes after payload", off);
  }
};

struct Writer {
  FILE* f = nullptr;
  std::string path;
  explicit Writer(const char* p) : path(p ? p : "") {
    HMI_CHECK(p != nullptr, HMI_CONFIG_ERROR, "null path");
    f = std::fopen(p, "wb");
    HMI_CHECK(f != nullptr, HMI_CONFIG_ERROR, "cannot open " + path + " for writing");
  }
  ~Writer() {
    if (f) std::fclose(f);
  }
  void bytes(const void* p, size_t n) {
    HMI_CHECK(n == 0 || std::fwrite(p, 1, n, f) == n, HMI_CONFIG_ERROR, "write failed for " + path);
  }
  void u32(uint32_t v) { bytes(&v, 4); }
  void u64(uint64_t v) { bytes(&v, 8); }
  void close() {
    const int rc = std::fclose(f);
    f = nullptr;
    HMI_CHECK(rc == 0, HMI_CONFIG_ERROR, "close failed for " + path);
  }
};

size_t layer_floats(size_t d, size_t f) { return 4 * (d * d + d) + (d * f + f) + (f * d + d) + 4 * d; }

template <typename F>
int ingest_guarded(F&& fn) {
  try {
    fn();
    return HMI_OK;
  } catch (const HmiError& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::bad_alloc& e) {
    set_last_error(std::string("host allocation failed: ") + e.what());
    return HMI_CAPACITY_ERROR;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return HMI_CUDA_ERROR;
  }
}

}  // namespace

// ADP1 body straight into `body` when the header matches the expected dimensions (one pass;
// the bulk registration path). Dimension mismatch -> DimensionError, format as hmi_adapter_set_load.
void load_adp1_expect(const char* path, uint32_t L, uint32_t D, uint32_t R, float* body) {
  Reader rd(path);
  rd.magic("ADP1");
  (void)rd.str();
  const uint32_t l = rd.u32(), d = rd.u32(), r = rd.u32();
  if (l == 0 || d == 0 || r == 0 || r >= d) rd.fail("adapter header dimensions invalid", rd.off);
  HMI_CHECK(l == L && d == D && r == R, HMI_DIMENSION_ERROR,
            std::string("adapter set in ") + path + " does not match the model");
  const size_t per = static_cast<size_t>(D) * R * 2 + R + D;
  rd.f32s(body, per * L);
  rd.expect_end();
}
}  // namespace hmi_b200

extern "C" {

// ---- PLT1 ---------------------------------------------------------------
int hmi_plot_table_load(const char* path, hmi_plot_table** out, uint32_t* version_id,
                        uint32_t* parent_id, uint32_t* alpha_centi) {
  using namespace hmi_b200;
  return ingest_guarded([&] {
    HMI_CHECK(out != nullptr, HMI_CONFIG_ERROR, "null argument");
    Reader r(path);
    r.magic("PLT1");
    const uint32_t version = r.u32();
    const uint32_t parent = r.u32();
    (void)r.str();  // domain label
    const uint32_t ngram = r.u32();
    const uint32_t d = r.u32();
    const uint32_t count = r.u32();
    const uint32_t alpha = r.u32();
    if (ngram == 0 || d == 0) r.fail("table header has zero ngram or hidden size", r.off);
    HMI_CHECK(ngram <= static_cast<uint32_t>(kMaxFragment), HMI_CONFIG_ERROR,
              "table n-gram order above 5 is not supported on the device");
    auto* t = new hmi_plot_table;
    try {
      t->ngram = ngram;
      t->d = d;
      t->key_len.reserve(count);
      t->keys.reserve(static_cast<size_t>(count) * ngram);
      t->freq.reserve(count);
      std::set<std::vector<uint32_t>> seen;
      for (uint32_t i = 0; i < count; ++i) {
        const size_t at = r.off;
        const uint32_t kl = r.u32();
        if (kl == 0 || kl > ngram)
          r.fail("entry key length " + std::to_string(kl) + " outside [1, " + std::to_string(ngram) + "]", at);
        std::vector<uint32_t> key(kl);
        for (uint32_t& x : key) x = r.u32();
        const uint64_t fr = r.u64();
        if (fr == 0) r.fail("entry frequency must be >= 1", at);
        const size_t base = t->reps.size();
        t->reps.resize(base + static_cast<size_t>(kl) * d);
        r.f32s(t->reps.data() + base, static_cast<size_t>(kl) * d);
        if (!seen.insert(key).second) r.fail("duplicate entry key", at);
        t->key_len.push_back(kl);
        for (uint32_t j = 0; j < ngram; ++j) t->keys.push_back(j < kl ? key[j] : 0);
        t->freq.push_back(fr);
      }
      r.expect_end();
    } catch (...) {
      delete t;
      throw;
    }
    if (version_id) *version_id = version;
    if (parent_id) *parent_id = parent;
    if (alpha_centi) *alpha_centi = alpha;
    *out = t;
  });
}

int hmi_plot_table_save(const hmi_plot_table* t, const char* path, uint32_t version_id,
                        uint32_t parent_id, const char* domain_label, uint32_t alpha_centi) {
  using namespace hmi_b200;
  return ingest_guarded([&] {
    HMI_CHECK(t != nullptr, HMI_CONFIG_ERROR, "null table");
    HMI_CHECK(!t->reps.empty() || t->key_len.empty(), HMI_CONFIG_ERROR,
              "table has no representations (a key selection only)");
    // entries in std::map key order (plot_io.cpp:25); tables from this library already are
    const uint32_t n = static_cast<uint32_t>(t->key_len.size());
    std::vector<uint32_t> order(n);
    std::vector<uint64_t> row0(n + 1, 0);
    for (uint32_t i = 0; i < n; ++i) {
      order[i] = i;
      row0[i + 1] = row0[i] + t->key_len[i];
    }
    auto key_of = [&](uint32_t i) {
      return std::vector<uint32_t>(t->keys.begin() + static_cast<size_t>(i) * t->ngram,
                                   t->keys.begin() + static_cast<size_t>(i) * t->ngram + t->key_len[i]);
    };
    std::stable_sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) { return key_of(a) < key_of(b); });
    Writer w(path);
    w.bytes("PLT1", 4);
    w.u32(version_id);
    w.u32(parent_id);
    const std::string label = domain_label ? domain_label : "";
    w.u32(static_cast<uint32_t>(label.size()));
    w.bytes(label.data(), label.size());
    w.u32(t->ngram);
    w.u32(t->d);
    w.u32(n);
    w.u32(alpha_centi);
    for (uint32_t i : order) {
      w.u32(t->key_len[i]);
      for (uint32_t j = 0; j < t->key_len[i]; ++j) w.u32(t->keys[static_cast<size_t>(i) * t->ngram + j]);
      w.u64(t->freq[i]);
      w.bytes(t->reps.data() + row0[i] * t->d, static_cast<size_t>(t->key_len[i]) * t->d * 4);
    }
    w.close();
  });
}

// ---- ADP1 ---------------------------------------------------------------
int hmi_adapter_set_load(const char* path, char* task_id, uint32_t task_id_cap, uint32_t* layers,
                         uint32_t* d, uint32_t* r, float* body) {
  using namespace hmi_b200;
  return ingest_guarded([&] {
    Reader rd(path);
    rd.magic("ADP1");
    const std::string id = rd.str();
    const uint32_t L = rd.u32(), D = rd.u32(), R = rd.u32();
    if (L == 0 || D == 0 || R == 0 || R >= D) rd.fail("adapter header dimensions invalid", rd.off);
    const size_t per = static_cast<size_t>(D) * R + R + static_cast<size_t>(R) * D + D;
    rd.f32s(body, per * L);  // W_down, b_down, W_up, b_up per layer (adapter_set.cpp:62-71)
    rd.expect_end();
    if (task_id && task_id_cap) {
      const size_t n = std::min<size_t>(id.size(), task_id_cap - 1);
      std::memcpy(task_id, id.data(), n);
      task_id[n] = '\0';
    }
    if (layers) *layers = L;
    if (d) *d = D;
    if (r) *r = R;
  });
}

// ---- HMI1 ---------------------------------------------------------------
int hmi_model_load(const char* path, hmi_model_config* cfg, float* token_emb, float* pos_emb,
                   float* lower_f32, float* higher_f32) {
  using namespace hmi_b200;
  return ingest_guarded([&] {
    HMI_CHECK(cfg != nullptr, HMI_CONFIG_ERROR, "null config");
    Reader rd(path);
    rd.magic("HMI1");
    hmi_model_config c{};
    c.hidden_size = rd.u32();
    c.heads = rd.u32();
    c.lower_layers = rd.u32();
    c.higher_layers = rd.u32();
    c.ffn_size = rd.u32();
    c.vocab_size = rd.u32();
    c.mode = rd.u32();
    c.max_fragment = rd.u32();
    c.seed = rd.u32();
    // ModelConfig::validate (weights.cpp)
    HMI_CHECK(c.hidden_size > 0 && c.heads > 0 && c.hidden_size % c.heads == 0, HMI_CONFIG_ERROR,
              "hidden_size must be a positive multiple of heads");
    HMI_CHECK(c.ffn_size > 0 && c.vocab_size > 0 && c.max_fragment > 0 && c.mode <= 1,
              HMI_CONFIG_ERROR, "model config fields invalid");
    const size_t d = c.hidden_size, lf = layer_floats(d, c.ffn_size);
    rd.f32s(token_emb, static_cast<size_t>(c.vocab_size) * d);
    rd.f32s(pos_emb, static_cast<size_t>(c.max_fragment) * d);
    rd.f32s(lower_f32, lf * c.lower_layers);
    rd.f32s(higher_f32, lf * c.higher_layers);
    rd.expect_end();
    *cfg = c;
  });
}

// ---- straight into a GPU context -------------------------------------------------
int hmi_gpu_upload_plot_table(hmi_gpu_ctx* ctx, uint32_t version_id, uint32_t parent_id,
                              const hmi_plot_table* t) {
  using namespace hmi_b200;
  if (t == nullptr) {
    set_last_error("null table");
    return HMI_CONFIG_ERROR;
  }
  if (t->reps.empty() && !t->key_len.empty()) {
    set_last_error("table has no representations (a key selection only)");
    return HMI_CONFIG_ERROR;
  }
  return hmi_gpu_upload_table(ctx, version_id, parent_id, static_cast<uint32_t>(t->key_len.size()),
                              t->key_len.data(), t->keys.data(), t->reps.data());
}

int hmi_gpu_register_task_file(hmi_gpu_ctx* ctx, uint32_t task_idx, const char* adp1_path) {
  using namespace hmi_b200;
  uint32_t L = 0, D = 0, R = 0;
  int rc = hmi_adapter_set_load(adp1_path, nullptr, 0, &L, &D, &R, nullptr);
  if (rc != HMI_OK) return rc;
  std::vector<float> body;
  try {
    body.resize((static_cast<size_t>(D) * R * 2 + R + D) * L);
  } catch (const std::bad_alloc&) {
    set_last_error("host allocation failed");
    return HMI_CAPACITY_ERROR;
  }
  rc = hmi_adapter_set_load(adp1_path, nullptr, 0, nullptr, nullptr, nullptr, body.data());
  if (rc != HMI_OK) return rc;
  // dimensions against the context: checked by hmi_gpu_register_task_dims
  rc = hmi_gpu_check_adapter_dims(ctx, L, D, R);
  if (rc != HMI_OK) return rc;
  return hmi_gpu_register_task(ctx, task_idx, body.data());
}

}  // extern "C"
