// SPDX-License-Identifier: Apache-2.0
//
// Seeded artefact generators of the serving API: identical values to the
// reference's generators, so a deployment (and bench.py) can materialise the
// same "random-init" hPLMs the reference would:
//   Xoshiro256pp            proj/include/hmi/rng.hpp:11-56
//   generate_model          proj/src/transformer/weights.cpp:72-88 (draw order :31-52)
//   generate_adapter_set    proj/src/adapters/adapter_set.cpp:15-25 (+ weights.cpp:90-103)
//   generate_output_head    proj/src/transformer/weights.cpp:105-118
// Bit-exactness against the reference is pinned by tests/test_generate.py.
#include <cstdint>
#include <cstring>
#include <vector>

#include "host_util.hpp"

namespace {

struct Xoshiro {
  uint64_t s[4];
  explicit Xoshiro(uint64_t seed) {
    uint64_t x = seed;
    for (auto& v : s) {
      x += 0x9e3779b97f4a7c15ULL;
      uint64_t z = x;
      z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
      z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
      v = z ^ (z >> 31);
    }
  }
  static uint64_t rotl(uint64_t v, int k) { return (v << k) | (v >> (64 - k)); }
  uint64_t next() {
    const uint64_t r = rotl(s[0] + s[3], 23) + s[0];
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl(s[3], 45);
    return r;
  }
  // uniform(-0.05, 0.05) as in rng.hpp:37-43, then base added and quantised to f32
  float draw(double base) {
    const double u = static_cast<double>(next() >> 11) * 0x1.0p-53;
    return static_cast<float>(base + (-0.05 + (0.05 - -0.05) * u));
  }
  void fill(float* out, size_t n, double base = 0.0) {
    for (size_t i = 0; i < n; ++i) {
      if (out) {
        out[i] = draw(base);
      } else {
        draw(base);
      }
    }
  }
};

void draw_layer(Xoshiro& g, size_t d, size_t f, float* w) {
  auto take = [&](size_t n, double base) {
    g.fill(w, n, base);
    if (w) w += n;
  };
  for (int i = 0; i < 4; ++i) {  // wq,bq,wk,bk,wv,bv,wo,bo
    take(d * d, 0.0);
    take(d, 0.0);
  }
  take(d * f, 0.0);  // w1
  take(f, 0.0);      // b1
  take(f * d, 0.0);  // w2
  take(d, 0.0);      // b2
  take(d, 1.0);      // ln1_gain
  take(d, 0.0);      // ln1_shift
  take(d, 1.0);      // ln2_gain
  take(d, 0.0);      // ln2_shift
}

}  // namespace

extern "C" {

// Writes the higher-stack weights (HMI1 per-layer order) of generate_model(cfg);
// tok_emb / pos_emb / lower may be NULL (their draws are consumed either way).
int hmi_generate_model(const hmi_model_config* c, float* tok_emb, float* pos_emb, float* lower,
                       float* higher) {
  if (!c || c->hidden_size == 0 || c->heads == 0 || c->hidden_size % c->heads != 0) {
    hmi_b200::set_last_error("hidden_size must be a positive multiple of heads");
    return HMI_CONFIG_ERROR;
  }
  Xoshiro g(c->seed);
  const size_t d = c->hidden_size, f = c->ffn_size;
  const size_t lf = 4 * (d * d + d) + (d * f + f) + (f * d + d) + 4 * d;
  g.fill(tok_emb, static_cast<size_t>(c->vocab_size) * d);
  g.fill(pos_emb, static_cast<size_t>(c->max_fragment) * d);
  for (uint32_t l = 0; l < c->lower_layers; ++l) draw_layer(g, d, f, lower ? lower + l * lf : nullptr);
  for (uint32_t l = 0; l < c->higher_layers; ++l) draw_layer(g, d, f, higher ? higher + l * lf : nullptr);
  return HMI_OK;
}

int hmi_generate_adapter(const hmi_model_config* c, uint32_t r, uint64_t seed, float* out) {
  if (!c || r == 0 || r >= c->hidden_size) {
    hmi_b200::set_last_error("adapter bottleneck must be in [1, hidden_size)");
    return HMI_CONFIG_ERROR;
  }
  Xoshiro g(seed);
  const size_t d = c->hidden_size;
  for (uint32_t l = 0; l < c->higher_layers; ++l) {
    g.fill(out, d * r); out += d * r;
    g.fill(out, r);     out += r;
    g.fill(out, r * d); out += r * d;
    g.fill(out, d);     out += d;
  }
  return HMI_OK;
}

int hmi_generate_head(uint32_t d, uint32_t labels, uint64_t seed, float* w, float* b) {
  if (labels < 1) {
    hmi_b200::set_last_error("output head needs at least one label");
    return HMI_CONFIG_ERROR;
  }
  Xoshiro g(seed);
  g.fill(w, static_cast<size_t>(d) * labels);
  g.fill(b, labels);
  return HMI_OK;
}

}  // extern "C"
