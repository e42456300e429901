/* SPDX-License-Identifier: Apache-2.0
 *
 * hmi_oracle.c — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference's hot path, used as the parity checker
 * for the B200 product. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load this library; the product never links it.
 *
 * Numeric contract: the reference's *scalar* KernelTable
 * (proj/src/tensor/kernels_scalar.cpp:11-48), compiled with -ffp-contract=off
 * (proj/CMakeLists.txt:14-18). Every loop below keeps the reference's operation
 * order, so results are bit-identical to the reference run with
 * HMI_KERNELS=scalar. That is pinned by tests/test_oracle_pin.py against the
 * compiled reference (oracle/_ref) and the committed fixtures in tests/golden/.
 *
 * Sections and the reference code each one restates:
 *   xoshiro256++ / splitmix64 ........ proj/include/hmi/rng.hpp:11-56
 *   generate_model / adapter / head ... proj/src/transformer/weights.cpp:13-118,
 *                                       proj/src/adapters/adapter_set.cpp:15-25
 *   gemm / add / relu / layer_norm .... proj/src/tensor/kernels_scalar.cpp:11-40,
 *                                       proj/src/tensor/ops.cpp:25-116
 *   attention / ffn / adapter / layer . proj/src/transformer/model.cpp:13-94
 *   apply_head / argmax ............... proj/src/transformer/model.cpp:120-171
 *   VersionTree::lookup ............... proj/src/plot/version_tree.cpp:47-79
 *   resolve_window / retrieve_sequence  proj/src/plot/retrieval.cpp:23-124
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_DIMENSION 1
#define ORC_VOCABULARY 2
#define ORC_ROUTING 5
#define ORC_CONFIG 6
#define ORC_BUILD 7

/* ------------------------------------------------------------------------ */
/* xoshiro256++ seeded by splitmix64 (rng.hpp:13-48)                         */
/* ------------------------------------------------------------------------ */
typedef struct {
  uint64_t s[4];
} orc_rng;

static uint64_t rotl64(uint64_t v, int k) { return (v << k) | (v >> (64 - k)); }

void orc_rng_seed(orc_rng* r, uint64_t seed) {
  uint64_t x = seed;
  for (int i = 0; i < 4; ++i) {
    x += 0x9e3779b97f4a7c15ULL;
    uint64_t z = x;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    r->s[i] = z ^ (z >> 31);
  }
}

uint64_t orc_rng_next(orc_rng* r) {
  uint64_t* s = r->s;
  const uint64_t result = rotl64(s[0] + s[3], 23) + s[0];
  const uint64_t t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = rotl64(s[3], 45);
  return result;
}

static double rng_uniform01(orc_rng* r) { return (double)(orc_rng_next(r) >> 11) * 0x1.0p-53; }
static double rng_uniform(orc_rng* r, double lo, double hi) {
  return lo + (hi - lo) * rng_uniform01(r);
}

/* weights.cpp:13-29: draw() quantises to f32; draw_vector adds `base` first
 * (base 0 reproduces draw() exactly since 0.0 + u == u). */
static void draw_n(orc_rng* r, float* out, size_t n, double base) {
  for (size_t i = 0; i < n; ++i) out[i] = (float)(base + rng_uniform(r, -0.05, 0.05));
}

typedef struct {
  uint32_t hidden_size, heads, lower_layers, higher_layers, ffn_size, vocab_size, mode,
      max_fragment, seed;
} orc_config; /* config.hpp:10-24, field order of the HMI1 header (model_io.cpp:71-82) */

/* floats per layer in HMI1 declaration order (weights.hpp:15-21) */
size_t orc_layer_floats(const orc_config* c) {
  const size_t d = c->hidden_size, f = c->ffn_size;
  return 4 * (d * d + d) + (d * f + f) + (f * d + d) + 4 * d;
}

/* draw_layer, weights.cpp:31-52 */
static void draw_layer(orc_rng* r, const orc_config* c, float* w) {
  const size_t d = c->hidden_size, f = c->ffn_size;
  for (int i = 0; i < 4; ++i) { /* wq,bq,wk,bk,wv,bv,wo,bo */
    draw_n(r, w, d * d, 0.0); /* draw_matrix == draw() each, same as base 0 */
    w += d * d;
    draw_n(r, w, d, 0.0);
    w += d;
  }
  draw_n(r, w, d * f, 0.0); w += d * f; /* w1 */
  draw_n(r, w, f, 0.0);     w += f;     /* b1 */
  draw_n(r, w, f * d, 0.0); w += f * d; /* w2 */
  draw_n(r, w, d, 0.0);     w += d;     /* b2 */
  draw_n(r, w, d, 1.0);     w += d;     /* ln1_gain */
  draw_n(r, w, d, 0.0);     w += d;     /* ln1_shift */
  draw_n(r, w, d, 1.0);     w += d;     /* ln2_gain */
  draw_n(r, w, d, 0.0);                 /* ln2_shift */
}

/* generate_model, weights.cpp:72-88. Any output pointer may be NULL to skip
 * storing (the draws still happen, keeping the stream aligned). */
int orc_generate_model(const orc_config* c, float* tok_emb, float* pos_emb, float* lower,
                       float* higher) {
  orc_rng r;
  orc_rng_seed(&r, c->seed);
  const size_t d = c->hidden_size;
  const size_t lf = orc_layer_floats(c);
  float* scratch = NULL;
  size_t big = (size_t)c->vocab_size * d;
  if (lf > big) big = lf;
  if (!tok_emb || !pos_emb || !lower || !higher) {
    scratch = (float*)malloc(big * sizeof(float));
    if (!scratch) return ORC_CONFIG;
  }
  draw_n(&r, tok_emb ? tok_emb : scratch, (size_t)c->vocab_size * d, 0.0);
  draw_n(&r, pos_emb ? pos_emb : scratch, (size_t)c->max_fragment * d, 0.0);
  for (uint32_t l = 0; l < c->lower_layers; ++l) draw_layer(&r, c, lower ? lower + l * lf : scratch);
  for (uint32_t l = 0; l < c->higher_layers; ++l)
    draw_layer(&r, c, higher ? higher + l * lf : scratch);
  free(scratch);
  return ORC_OK;
}

size_t orc_adapter_layer_floats(uint32_t d, uint32_t r) { return (size_t)d * r + r + (size_t)r * d + d; }

/* generate_adapter_set (adapter_set.cpp:15-25) -> generate_adapter_params (weights.cpp:90-103) */
int orc_generate_adapter(const orc_config* c, uint32_t r, uint64_t seed, float* out) {
  if (r == 0 || r >= c->hidden_size) return ORC_CONFIG;
  orc_rng g;
  orc_rng_seed(&g, seed);
  const size_t d = c->hidden_size;
  for (uint32_t l = 0; l < c->higher_layers; ++l) {
    draw_n(&g, out, d * r, 0.0); out += d * r;
    draw_n(&g, out, r, 0.0);     out += r;
    draw_n(&g, out, r * d, 0.0); out += r * d;
    draw_n(&g, out, d, 0.0);     out += d;
  }
  return ORC_OK;
}

/* generate_output_head, weights.cpp:105-118 */
int orc_generate_head(uint32_t d, uint32_t labels, uint64_t seed, float* w, float* b) {
  if (labels < 1) return ORC_CONFIG;
  orc_rng g;
  orc_rng_seed(&g, seed);
  draw_n(&g, w, (size_t)d * labels, 0.0);
  draw_n(&g, b, labels, 0.0);
  return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* dense ops (kernels_scalar.cpp:11-40, ops.cpp:25-131)                      */
/* ------------------------------------------------------------------------ */
/* c = a . b with b given as f32 (weights are f32-exact doubles in the reference) */
static void gemm_f32w(const double* a, const float* b, double* c, size_t m, size_t k, size_t n) {
  for (size_t i = 0; i < m; ++i) {
    double* crow = c + i * n;
    for (size_t j = 0; j < n; ++j) crow[j] = 0.0;
    for (size_t p = 0; p < k; ++p) {
      const double aip = 1.0 * a[i * k + p];
      const float* brow = b + p * n;
      for (size_t j = 0; j < n; ++j) crow[j] += aip * (double)brow[j];
    }
  }
}

static void add_bias(double* x, const float* bias, size_t rows, size_t cols) {
  for (size_t r = 0; r < rows; ++r)
    for (size_t j = 0; j < cols; ++j) x[r * cols + j] = x[r * cols + j] + (double)bias[j];
}

static void relu(double* x, size_t n) {
  for (size_t i = 0; i < n; ++i)
    if (x[i] < 0.0) x[i] = 0.0;
}

static void add_inplace(double* x, const double* y, size_t n) {
  for (size_t i = 0; i < n; ++i) x[i] = x[i] + y[i];
}

/* layer_norm, ops.cpp:92-116 (epsilon 1e-5, ops.hpp:10) */
static void layer_norm(const double* x, const float* gain, const float* shift, double* out,
                       size_t rows, size_t n) {
  for (size_t r = 0; r < rows; ++r) {
    const double* row = x + r * n;
    double mean = 0.0;
    for (size_t j = 0; j < n; ++j) mean += row[j];
    mean /= (double)n;
    double var = 0.0;
    for (size_t j = 0; j < n; ++j) {
      const double dd = row[j] - mean;
      var += dd * dd;
    }
    var /= (double)n;
    const double inv = 1.0 / sqrt(var + 1e-5);
    double* orow = out + r * n;
    for (size_t j = 0; j < n; ++j) orow[j] = (row[j] - mean) * inv * (double)gain[j] + (double)shift[j];
  }
}

typedef struct {
  const float *wq, *bq, *wk, *bk, *wv, *bv, *wo, *bo, *w1, *b1, *w2, *b2, *ln1g, *ln1b, *ln2g, *ln2b;
} layer_view;

static layer_view view_layer(const float* w, size_t d, size_t f) {
  layer_view v;
  v.wq = w; w += d * d; v.bq = w; w += d;
  v.wk = w; w += d * d; v.bk = w; w += d;
  v.wv = w; w += d * d; v.bv = w; w += d;
  v.wo = w; w += d * d; v.bo = w; w += d;
  v.w1 = w; w += d * f; v.b1 = w; w += f;
  v.w2 = w; w += f * d; v.b2 = w; w += d;
  v.ln1g = w; w += d; v.ln1b = w; w += d;
  v.ln2g = w; w += d; v.ln2b = w;
  return v;
}

/* attention, model.cpp:26-76 (out = ctx.Wo + bo, len x d) */
static void attention(const double* h, const layer_view* w, const orc_config* c, size_t len,
                      size_t valid_len, double* out) {
  const size_t d = c->hidden_size;
  if (valid_len > len) valid_len = len;
  double* q = (double*)malloc(len * d * sizeof(double));
  double* k = (double*)malloc(len * d * sizeof(double));
  double* v = (double*)malloc(len * d * sizeof(double));
  double* ctx = (double*)calloc(len * d, sizeof(double));
  double* probs = (double*)malloc(len * sizeof(double));
  gemm_f32w(h, w->wq, q, len, d, d); add_bias(q, w->bq, len, d);
  gemm_f32w(h, w->wk, k, len, d, d); add_bias(k, w->bk, len, d);
  gemm_f32w(h, w->wv, v, len, d, d); add_bias(v, w->bv, len, d);
  const size_t heads = c->heads, dh = d / heads;
  const double scale = 1.0 / sqrt((double)dh);
  for (size_t g = 0; g < heads; ++g) {
    const size_t off = g * dh;
    for (size_t i = 0; i < len; ++i) {
      const size_t limit = c->mode == 1 ? i + 1 : valid_len;
      double mx = -INFINITY;
      for (size_t j = 0; j < limit; ++j) {
        double s = 0.0;
        for (size_t cc = 0; cc < dh; ++cc) s += q[i * d + off + cc] * k[j * d + off + cc];
        probs[j] = s * scale;
        mx = probs[j] > mx ? probs[j] : mx; /* std::max(mx, probs[j]) */
      }
      double sum = 0.0;
      for (size_t j = 0; j < limit; ++j) {
        probs[j] = exp(probs[j] - mx);
        sum += probs[j];
      }
      for (size_t cc = 0; cc < dh; ++cc) {
        double acc = 0.0;
        for (size_t j = 0; j < limit; ++j) acc += probs[j] * v[j * d + off + cc];
        ctx[i * d + off + cc] = acc / sum;
      }
    }
  }
  gemm_f32w(ctx, w->wo, out, len, d, d);
  add_bias(out, w->bo, len, d);
  free(q); free(k); free(v); free(ctx); free(probs);
}

/* adapter_apply, model.cpp:13-24: up(relu(down(a)+bd))+bu + a (in place on a) */
static void adapter_apply(double* a, const float* ad, size_t len, size_t d, size_t r) {
  const float* wd = ad;
  const float* bd = wd + d * r;
  const float* wu = bd + r;
  const float* bu = wu + r * d;
  double* mid = (double*)malloc(len * r * sizeof(double));
  double* out = (double*)malloc(len * d * sizeof(double));
  gemm_f32w(a, wd, mid, len, d, r);
  add_bias(mid, bd, len, r);
  relu(mid, len * r);
  gemm_f32w(mid, wu, out, len, r, d);
  add_bias(out, bu, len, d);
  add_inplace(out, a, len * d);
  memcpy(a, out, len * d * sizeof(double));
  free(mid); free(out);
}

/* layer_forward, model.cpp:84-94 (in place on h) */
static void layer_forward(double* h, const float* lw, const float* adapter, uint32_t r,
                          const orc_config* c, size_t len, size_t valid_len) {
  const size_t d = c->hidden_size, f = c->ffn_size;
  layer_view w = view_layer(lw, d, f);
  double* attn = (double*)malloc(len * d * sizeof(double));
  double* x = (double*)malloc(len * d * sizeof(double));
  double* mid = (double*)malloc(len * f * sizeof(double));
  double* ff = (double*)malloc(len * d * sizeof(double));
  attention(h, &w, c, len, valid_len, attn);
  if (adapter) adapter_apply(attn, adapter, len, d, r);
  add_inplace(attn, h, len * d); /* add(attn, h): attn + h */
  layer_norm(attn, w.ln1g, w.ln1b, x, len, d);
  gemm_f32w(x, w.w1, mid, len, d, f);
  add_bias(mid, w.b1, len, f);
  relu(mid, len * f);
  gemm_f32w(mid, w.w2, ff, len, f, d);
  add_bias(ff, w.b2, len, d);
  /* add(x, f) = x + f, then LN2 */
  for (size_t i = 0; i < len * d; ++i) attn[i] = x[i] + ff[i];
  layer_norm(attn, w.ln2g, w.ln2b, h, len, d);
  free(attn); free(x); free(mid); free(ff);
}

static int argmax(const double* v, size_t n) {
  int best = 0;
  for (size_t i = 1; i < n; ++i)
    if (v[i] > v[best]) best = (int)i;
  return best;
}

/* project_row, model.cpp:130-136 */
static void project_row(const double* h, size_t row, size_t d, const float* hw, const float* hb,
                        uint32_t labels, double* scores) {
  gemm_f32w(h + row * d, hw, scores, 1, d, labels);
  add_bias(scores, hb, 1, labels);
}

/* Runs the higher stack (model.cpp:173-185) over h [len x d] in place using
 * layer_forward with valid_len (the batched stage_compute contract, SPEC.md:461-469:
 * keys at or beyond valid_len are never read), then apply_head (model.cpp:140-171).
 *   adapters: higher_layers x adapter_layer_floats, or NULL (no adapters)
 *   head_kind: 0 cls (row 0), 1 token_tag (rows < valid_len), 2 lm (row valid_len-1)
 *   scores:    labels doubles (cls/lm); tags: valid_len ints (token_tag)
 */
int orc_higher_forward(const orc_config* c, const float* higher, double* h, size_t len,
                       size_t valid_len, const float* adapters, uint32_t r, const float* head_w,
                       const float* head_b, uint32_t labels, int head_kind, double* scores,
                       int32_t* label, int32_t* tags) {
  if (len == 0 || valid_len == 0) return ORC_DIMENSION;
  if (valid_len > len) valid_len = len;
  const size_t lf = orc_layer_floats(c);
  const size_t af = orc_adapter_layer_floats(c->hidden_size, r);
  for (uint32_t l = 0; l < c->higher_layers; ++l) {
    layer_forward(h, higher + l * lf, adapters ? adapters + l * af : NULL, r, c, len, valid_len);
  }
  const size_t d = c->hidden_size;
  if (head_kind == 0 || head_kind == 2) {
    const size_t row = head_kind == 0 ? 0 : valid_len - 1;
    project_row(h, row, d, head_w, head_b, labels, scores);
    *label = argmax(scores, labels);
  } else {
    double* tmp = (double*)malloc(labels * sizeof(double));
    for (size_t i = 0; i < valid_len; ++i) {
      project_row(h, i, d, head_w, head_b, labels, tmp);
      tags[i] = argmax(tmp, labels);
    }
    free(tmp);
  }
  return ORC_OK;
}

/*
 * lower_stack_forward, model.cpp:96-118: h[i] = token_emb[t_i] + position_emb[i] (fragment-local
 * positions), then every lower layer (layer_forward without an adapter, all keys valid).
 *   tok_emb [vocab x d], pos_emb [max_fragment x d], lower = lower_layers x layer_floats
 *   out [len x d] doubles (the PLOT rep of the fragment)
 */
int orc_lower_forward(const orc_config* c, const float* tok_emb, const float* pos_emb,
                      const float* lower, const uint32_t* tokens, size_t len, double* out) {
  if (len == 0 || len > c->max_fragment) return ORC_DIMENSION;
  const size_t d = c->hidden_size;
  for (size_t i = 0; i < len; ++i) {
    if (tokens[i] >= c->vocab_size) return ORC_VOCABULARY;
    for (size_t j = 0; j < d; ++j) {
      out[i * d + j] = (double)tok_emb[(size_t)tokens[i] * d + j] + (double)pos_emb[i * d + j];
    }
  }
  const size_t lf = orc_layer_floats(c);
  for (uint32_t l = 0; l < c->lower_layers; ++l) {
    layer_forward(out, lower + l * lf, NULL, 0, c, len, len);
  }
  return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* PLOT version tree + retrieval                                             */
/* ------------------------------------------------------------------------ */
/* Tables are uploaded as arrays: entry e has key_len[e] tokens in
 * keys[e*ngram ...] and key_len[e] rep rows. Rep rows of all tables are
 * numbered globally in upload order (table order, entry order, row order);
 * that global row id is the "gather index" the device must reproduce. */
typedef struct {
  uint64_t h;
  uint32_t entry;
  uint32_t used;
} slot_t;

typedef struct {
  uint32_t version_id, parent_id; /* parent 0xffffffff = root */
  uint32_t n;
  uint32_t* key_len;
  uint32_t* keys;      /* n x ngram */
  uint64_t* row_base;  /* global row id of the entry's first row */
  slot_t* hash;
  uint64_t hcap;
} orc_table;

typedef struct {
  uint32_t ngram, d;
  uint32_t ntables;
  orc_table* tables;
  uint64_t nrows;
  float* reps; /* nrows x d */
} orc_tree;

static uint64_t key_hash(const uint32_t* k, uint32_t len) {
  uint64_t h = 1469598103934665603ULL ^ len;
  for (uint32_t i = 0; i < len; ++i) {
    h ^= k[i];
    h *= 1099511628211ULL;
    h ^= h >> 29;
  }
  return h;
}

void* orc_tree_create(uint32_t ngram, uint32_t d) {
  orc_tree* t = (orc_tree*)calloc(1, sizeof(orc_tree));
  t->ngram = ngram;
  t->d = d;
  return t;
}

void orc_tree_destroy(void* p) {
  orc_tree* t = (orc_tree*)p;
  if (!t) return;
  for (uint32_t i = 0; i < t->ntables; ++i) {
    free(t->tables[i].key_len); free(t->tables[i].keys); free(t->tables[i].row_base);
    free(t->tables[i].hash);
  }
  free(t->tables);
  free(t->reps);
  free(t);
}

static orc_table* find_table(orc_tree* t, uint32_t version) {
  for (uint32_t i = 0; i < t->ntables; ++i)
    if (t->tables[i].version_id == version) return &t->tables[i];
  return NULL;
}

/* Adds one table (root: parent 0xffffffff). Mirrors VersionTree::add_branch's
 * parent check (version_tree.cpp:17-30). */
int orc_tree_add_table(void* p, uint32_t version_id, uint32_t parent_id, uint32_t n,
                       const uint32_t* key_len, const uint32_t* keys, const float* reps) {
  orc_tree* t = (orc_tree*)p;
  if (parent_id != 0xffffffffu && !find_table(t, parent_id)) return ORC_ROUTING;
  t->tables = (orc_table*)realloc(t->tables, (t->ntables + 1) * sizeof(orc_table));
  orc_table* tb = &t->tables[t->ntables++];
  memset(tb, 0, sizeof(*tb));
  tb->version_id = version_id;
  tb->parent_id = parent_id;
  tb->n = n;
  tb->key_len = (uint32_t*)malloc((n ? n : 1) * sizeof(uint32_t));
  tb->keys = (uint32_t*)malloc((n ? n : 1) * (size_t)t->ngram * sizeof(uint32_t));
  tb->row_base = (uint64_t*)malloc((n ? n : 1) * sizeof(uint64_t));
  memcpy(tb->key_len, key_len, n * sizeof(uint32_t));
  memcpy(tb->keys, keys, (size_t)n * t->ngram * sizeof(uint32_t));
  uint64_t rows = 0;
  for (uint32_t e = 0; e < n; ++e) {
    if (key_len[e] == 0 || key_len[e] > t->ngram) return ORC_DIMENSION;
    tb->row_base[e] = t->nrows + rows;
    rows += key_len[e];
  }
  t->reps = (float*)realloc(t->reps, (t->nrows + rows) * (size_t)t->d * sizeof(float));
  memcpy(t->reps + t->nrows * t->d, reps, rows * (size_t)t->d * sizeof(float));
  t->nrows += rows;
  tb->hcap = 16;
  while (tb->hcap < 2ull * n) tb->hcap <<= 1;
  tb->hash = (slot_t*)calloc(tb->hcap, sizeof(slot_t));
  for (uint32_t e = 0; e < n; ++e) {
    const uint32_t* k = tb->keys + (size_t)e * t->ngram;
    uint64_t h = key_hash(k, key_len[e]);
    for (uint64_t i = h & (tb->hcap - 1);; i = (i + 1) & (tb->hcap - 1)) {
      if (!tb->hash[i].used) {
        tb->hash[i].used = 1; tb->hash[i].h = h; tb->hash[i].entry = e;
        break;
      }
      const uint32_t oe = tb->hash[i].entry;
      if (tb->key_len[oe] == key_len[e] &&
          memcmp(tb->keys + (size_t)oe * t->ngram, k, key_len[e] * sizeof(uint32_t)) == 0)
        return ORC_BUILD; /* duplicate key */
    }
  }
  return ORC_OK;
}

static int table_find(const orc_tree* t, const orc_table* tb, const uint32_t* k, uint32_t len) {
  if (tb->n == 0) return -1;
  uint64_t h = key_hash(k, len);
  for (uint64_t i = h & (tb->hcap - 1);; i = (i + 1) & (tb->hcap - 1)) {
    if (!tb->hash[i].used) return -1;
    const uint32_t e = tb->hash[i].entry;
    if (tb->hash[i].h == h && tb->key_len[e] == len &&
        memcmp(tb->keys + (size_t)e * t->ngram, k, len * sizeof(uint32_t)) == 0)
      return (int)e;
  }
}

/* VersionTree::lookup (version_tree.cpp:47-79): branch table first, then the
 * parent chain to the root. Returns the global row id of the entry's first row
 * or -1; *src_version receives the answering table's version id. */
static int64_t tree_lookup(orc_tree* t, uint32_t version, const uint32_t* k, uint32_t len,
                           uint32_t* src_version) {
  orc_table* tb = find_table(t, version);
  while (tb) {
    int e = table_find(t, tb, k, len);
    if (e >= 0) {
      *src_version = tb->version_id;
      return (int64_t)tb->row_base[e];
    }
    if (tb->parent_id == 0xffffffffu) break;
    tb = find_table(t, tb->parent_id);
  }
  return -1;
}

/* resolve_window (retrieval.cpp:23-69). For each position p of the window:
 * longest stored sub-gram containing p, leftmost among equals. Writes the
 * global row id and the level (sub-gram length) per position. */
static int resolve_window(orc_tree* t, uint32_t version, const uint32_t* tok, uint32_t len,
                          int64_t* rows, uint32_t* levels, uint32_t* srcs) {
  int64_t memo[8][8];
  uint32_t memo_src[8][8];
  int memo_set[8][8];
  memset(memo_set, 0, sizeof(memo_set));
  for (uint32_t p = 0; p < len; ++p) {
    int resolved = 0;
    for (uint32_t k = len; k >= 1 && !resolved; --k) {
      const uint32_t o_lo = p + 1 >= k ? p + 1 - k : 0;
      const uint32_t o_hi = p < len - k ? p : len - k;
      for (uint32_t o = o_lo; o <= o_hi; ++o) {
        if (!memo_set[o][k]) {
          memo[o][k] = tree_lookup(t, version, tok + o, k, &memo_src[o][k]);
          memo_set[o][k] = 1;
        }
        if (memo[o][k] >= 0) {
          rows[p] = memo[o][k] + (p - o);
          levels[p] = k;
          srcs[p] = memo_src[o][k];
          resolved = 1;
          break;
        }
      }
    }
    if (!resolved) return ORC_BUILD; /* uni-gram backstop missing */
  }
  return ORC_OK;
}

/* retrieve_sequence (retrieval.cpp:82-124).
 *   out    : len x d doubles (bit-identical to the reference)
 *   gather : len x ngram int64 — for position p, the global rep row taken from
 *            the k-th window covering p in ascending window order (-1 unused)
 *   levels : len x ngram sub-gram lengths (0 unused)
 * Encoder windows are centred (hl = (n-1)/2 left, hr = n-1-hl right) and clipped;
 * causal position i takes row i-start of the window [max(0, i-n+1), i]. */
int orc_retrieve(void* p, uint32_t version, const uint32_t* tokens, uint32_t len, int mode,
                 double* out, int64_t* gather, uint32_t* levels, uint32_t* srcs) {
  orc_tree* t = (orc_tree*)p;
  if (len == 0) return ORC_DIMENSION;
  if (!find_table(t, version)) return ORC_ROUTING;
  const uint32_t n = t->ngram, d = t->d;
  int64_t wrows[8];
  uint32_t wlev[8], wsrc[8];
  for (size_t i = 0; i < (size_t)len * n; ++i) {
    if (gather) gather[i] = -1;
    if (levels) levels[i] = 0;
    if (srcs) srcs[i] = 0xffffffffu;
  }
  if (mode == 1) {
    for (uint32_t i = 0; i < len; ++i) {
      const uint32_t start = i + 1 >= n ? i + 1 - n : 0;
      int rc = resolve_window(t, version, tokens + start, i - start + 1, wrows, wlev, wsrc);
      if (rc) return rc;
      const int64_t row = wrows[i - start];
      for (uint32_t j = 0; j < d; ++j) out[(size_t)i * d + j] = (double)t->reps[row * d + j];
      if (gather) gather[(size_t)i * n] = row;
      if (levels) levels[(size_t)i * n] = wlev[i - start];
      if (srcs) srcs[(size_t)i * n] = wsrc[i - start];
    }
    return ORC_OK;
  }
  const uint32_t hl = (n - 1) / 2, hr = n - 1 - hl;
  uint32_t* counts = (uint32_t*)calloc(len, sizeof(uint32_t));
  memset(out, 0, (size_t)len * d * sizeof(double));
  for (uint32_t c = 0; c < len; ++c) {
    const uint32_t start = c >= hl ? c - hl : 0;
    const uint32_t end = (c + hr < len - 1) ? c + hr : len - 1;
    int rc = resolve_window(t, version, tokens + start, end - start + 1, wrows, wlev, wsrc);
    if (rc) { free(counts); return rc; }
    for (uint32_t q = start; q <= end; ++q) {
      const int64_t row = wrows[q - start];
      double* o = out + (size_t)q * d;
      for (uint32_t j = 0; j < d; ++j) o[j] = o[j] + (double)t->reps[row * d + j];
      if (gather) gather[(size_t)q * n + counts[q]] = row;
      if (levels) levels[(size_t)q * n + counts[q]] = wlev[q - start];
      if (srcs) srcs[(size_t)q * n + counts[q]] = wsrc[q - start];
      counts[q] += 1;
    }
  }
  for (uint32_t q = 0; q < len; ++q) {
    const double inv = 1.0 / (double)counts[q];
    for (uint32_t j = 0; j < d; ++j) out[(size_t)q * d + j] *= inv;
  }
  free(counts);
  return ORC_OK;
}

/* Convenience: one request end to end = retrieve_sequence + higher stack + head
 * (the SPEC's bypass oracle). h is padded to `len` = max length of
 * the batch with zero rows beyond valid_len exactly as stage_compute pads. */
int orc_infer_one(const orc_config* c, const float* higher, void* tree, uint32_t version,
                  const uint32_t* tokens, uint32_t valid_len, uint32_t padded_len,
                  const float* adapters, uint32_t r, const float* head_w, const float* head_b,
                  uint32_t labels, int head_kind, double* scores, int32_t* label,
                  int32_t* tags) {
  const size_t d = c->hidden_size;
  if (padded_len < valid_len) padded_len = valid_len;
  double* h = (double*)calloc((size_t)padded_len * d, sizeof(double));
  int rc = orc_retrieve(tree, version, tokens, valid_len, (int)c->mode, h, NULL, NULL, NULL);
  if (rc == ORC_OK)
    rc = orc_higher_forward(c, higher, h, padded_len, valid_len, adapters, r, head_w, head_b,
                            labels, head_kind, scores, label, tags);
  free(h);
  return rc;
}
