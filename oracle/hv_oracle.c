/*
 * hv_oracle.c — plain-C restatement of the reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see hv_oracle.h). Parity pinned against golden
 * vectors produced by the reference library (tests/golden/).
 *
 * Every function cites the reference file:line it restates; paths are
 * relative to /root/reference/proj/. The model/encode paths restate the
 * reference's own byte-per-bit oracle (src/reference.cpp) rather than its
 * packed implementation, so a packing bug cannot be shared with the CUDA
 * engine; RNG and codebook generation restate the packed generators
 * (src/encoding.cpp) because their output format *is* packed words.
 *
 * Build: oracle/Makefile (gcc -O2 -ffp-contract=off — the reference is built
 * without FMA contraction on x86-64, so neither is this).
 */
#include "hv_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ======================================================================= */
/* RNG: std::mt19937_64 + splitmix64 substreams (rng.hpp:13-51).           */
/* mt19937_64 is fixed by the C++ standard ([rand.predef]): w=64, n=312,    */
/* m=156, r=31, a=0xB5026F5AA96619E9, u=29 d=0x5555555555555555, s=17       */
/* b=0x71D67FFFEDA60000, t=37 c=0xFFF7EEE000000000, l=43, f=6364136223846793005. */
/* ======================================================================= */

enum { MT_N = 312, MT_M = 156 };

/* rng.hpp:14-19 */
uint64_t hvo_splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

/* rng.hpp:22-24 */
uint64_t hvo_derive_seed(uint64_t seed, uint64_t tag) {
  return hvo_splitmix64(hvo_splitmix64(seed) ^ hvo_splitmix64(tag));
}

/* rng.hpp:30 (Rng(seed) : engine_(seed)) */
void hvo_rng_seed(hvo_rng* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < MT_N; ++i) {
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  }
  r->idx = MT_N;
}

static void mt_twist(hvo_rng* r) {
  const uint64_t upper = 0xFFFFFFFF80000000ULL; /* top w-r = 33 bits */
  const uint64_t lower = 0x7FFFFFFFULL;         /* low r = 31 bits */
  for (int i = 0; i < MT_N; ++i) {
    const uint64_t x = (r->mt[i] & upper) | (r->mt[(i + 1) % MT_N] & lower);
    uint64_t xa = x >> 1;
    if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
    r->mt[i] = r->mt[(i + MT_M) % MT_N] ^ xa;
  }
  r->idx = 0;
}

/* rng.hpp:32 next_u64 = engine_() */
uint64_t hvo_rng_next_u64(hvo_rng* r) {
  if (r->idx >= MT_N) mt_twist(r);
  uint64_t y = r->mt[r->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

/* rng.hpp:34-35: low 32 bits of one draw */
uint32_t hvo_rng_next_u32(hvo_rng* r) { return (uint32_t)hvo_rng_next_u64(r); }

/* rng.hpp:37-42: rejection sampling below 2^64 mod bound */
uint64_t hvo_rng_uniform_below(hvo_rng* r, uint64_t bound) {
  const uint64_t min = (0 - bound) % bound;
  uint64_t v = hvo_rng_next_u64(r);
  while (v < min) v = hvo_rng_next_u64(r);
  return v % bound;
}

/* rng.hpp:45-47 */
double hvo_rng_next_unit(hvo_rng* r) {
  return (double)(hvo_rng_next_u64(r) >> 11) * 0x1.0p-53;
}

void hvo_mt64_stream(uint64_t seed, size_t n, uint64_t* out) {
  hvo_rng r;
  hvo_rng_seed(&r, seed);
  for (size_t i = 0; i < n; ++i) out[i] = hvo_rng_next_u64(&r);
}

/* ======================================================================= */
/* Packed helpers (bitmat.hpp:30-86)                                       */
/* ======================================================================= */

/* bitmat.hpp:30-32 */
size_t hvo_words_per_row(size_t dim) { return (dim + 31) / 32; }

/* bitmat.hpp:64-67 */
static uint32_t padding_mask(size_t dim) {
  const size_t rem = dim % 32;
  return rem == 0 ? 0u : ~((1u << rem) - 1u);
}

/* bitmat.hpp:80-86 */
static void mask_padding(uint32_t* words, size_t rows, size_t dim) {
  const size_t w = hvo_words_per_row(dim);
  const uint32_t mask = padding_mask(dim);
  if (mask == 0 || w == 0) return;
  for (size_t r = 0; r < rows; ++r) words[r * w + w - 1] &= ~mask;
}

static int pbit(const uint32_t* row, size_t j) { return (int)((row[j / 32] >> (j % 32)) & 1u); }
static void pset(uint32_t* row, size_t j, int v) {
  const uint32_t m = 1u << (j % 32);
  if (v) row[j / 32] |= m; else row[j / 32] &= ~m;
}

/* kernels.cpp:201-216 restated bit by bit (exactly the same mapping) */
static void copy_bits(const uint32_t* src, size_t src_off, uint32_t* dst, size_t dst_off,
                      size_t len) {
  for (size_t k = 0; k < len; ++k) pset(dst, dst_off + k, pbit(src, src_off + k));
}

/* ======================================================================= */
/* Codebook generators (encoding.cpp:25-28, 156-255)                       */
/* ======================================================================= */

/* encoding.cpp:25-28 fill_random: one engine draw per word, low 32 bits */
static void fill_random(uint32_t* words, size_t rows, size_t dim, hvo_rng* r) {
  const size_t n = rows * hvo_words_per_row(dim);
  for (size_t i = 0; i < n; ++i) words[i] = hvo_rng_next_u32(r);
  mask_padding(words, rows, dim);
}

/* encoding.cpp:156-161 */
void hvo_generate_random(size_t count, size_t dim, uint64_t seed, uint32_t* out) {
  hvo_rng r;
  hvo_rng_seed(&r, seed);
  fill_random(out, count, dim, &r);
}

/* encoding.cpp:163-197 */
int hvo_generate_scale_random(size_t bins, size_t dim, uint64_t seed, uint32_t* out) {
  if (bins < 2) return HVO_INVALID_ARGUMENT;
  const size_t quota = dim / (2 * (bins - 1));
  if (quota == 0) return HVO_INVALID_ARGUMENT;
  const size_t w = hvo_words_per_row(dim);
  memset(out, 0, bins * w * sizeof(uint32_t));
  hvo_rng r;
  hvo_rng_seed(&r, seed);
  fill_random(out, 1, dim, &r); /* row 0 from a 1 x D fill (:175-179) */
  size_t* pool = (size_t*)malloc((dim ? dim : 1) * sizeof(size_t));
  for (size_t i = 0; i < dim; ++i) pool[i] = i;
  size_t remaining = dim;
  for (size_t k = 1; k < bins; ++k) {
    memcpy(out + k * w, out + (k - 1) * w, w * sizeof(uint32_t));
    for (size_t i = 0; i < quota; ++i) {
      const size_t idx = (size_t)hvo_rng_uniform_below(&r, remaining);
      const size_t pos = pool[idx];
      pool[idx] = pool[remaining - 1];
      --remaining;
      pset(out + k * w, pos, !pbit(out + k * w, pos));
    }
  }
  free(pool);
  return HVO_OK;
}

/* encoding.cpp:199-226 */
int hvo_generate_sandwich(size_t bins, size_t dim, uint64_t seed, uint32_t* out) {
  if (bins < 2) return HVO_INVALID_ARGUMENT;
  if (dim % 2 != 0) return HVO_INVALID_ARGUMENT;
  const size_t w = hvo_words_per_row(dim);
  memset(out, 0, bins * w * sizeof(uint32_t));
  hvo_rng r;
  hvo_rng_seed(&r, seed);
  for (size_t k = 0; k < bins; k += 2) fill_random(out + k * w, 1, dim, &r);
  const size_t half = dim / 2;
  uint32_t* tail = (uint32_t*)calloc(hvo_words_per_row(half) + 1, sizeof(uint32_t));
  for (size_t k = 1; k < bins; k += 2) {
    copy_bits(out + (k - 1) * w, 0, out + k * w, 0, half);
    if (k + 1 < bins) {
      copy_bits(out + (k + 1) * w, half, out + k * w, half, half);
    } else {
      fill_random(tail, 1, half, &r); /* fresh 1 x D/2 draw (:217-219) */
      copy_bits(tail, 0, out + k * w, half, half);
    }
  }
  free(tail);
  return HVO_OK;
}

/* encoding.cpp:228-255 (ID seed tag 1, Value seed tag 2) */
int hvo_make_codebook(int generation, size_t features, size_t bins, size_t dim, uint64_t seed,
                      uint32_t* id_out, uint32_t* value_out) {
  if (features == 0 || dim == 0) return HVO_INVALID_ARGUMENT;
  if (bins < 2) return HVO_INVALID_ARGUMENT;
  hvo_generate_random(features, dim, hvo_derive_seed(seed, 1), id_out);
  const uint64_t vseed = hvo_derive_seed(seed, 2);
  switch (generation) {
    case HVO_GEN_RANDOM: hvo_generate_random(bins, dim, vseed, value_out); return HVO_OK;
    case HVO_GEN_SCALE_RANDOM: return hvo_generate_scale_random(bins, dim, vseed, value_out);
    case HVO_GEN_SANDWICH: return hvo_generate_sandwich(bins, dim, vseed, value_out);
  }
  return HVO_INVALID_ARGUMENT;
}

/* ======================================================================= */
/* pack / unpack (kernels.cpp:44-73)                                       */
/* ======================================================================= */

long long hvo_pack(const uint8_t* dense, size_t rows, size_t dim, uint32_t* out) {
  for (size_t i = 0; i < rows * dim; ++i) {
    if (dense[i] > 1) return (long long)i; /* :45-51 */
  }
  const size_t w = hvo_words_per_row(dim);
  memset(out, 0, rows * w * sizeof(uint32_t));
  for (size_t r = 0; r < rows; ++r) {
    for (size_t j = 0; j < dim; ++j) out[r * w + j / 32] |= (uint32_t)dense[r * dim + j] << (j % 32);
  }
  return -1;
}

void hvo_unpack(const uint32_t* words, size_t rows, size_t dim, uint8_t* out) {
  const size_t w = hvo_words_per_row(dim);
  for (size_t r = 0; r < rows; ++r) {
    for (size_t j = 0; j < dim; ++j) out[r * dim + j] = (uint8_t)((words[r * w + j / 32] >> (j % 32)) & 1u);
  }
}

/* ======================================================================= */
/* Byte-per-bit kernels (reference.cpp:77-155)                            */
/* ======================================================================= */

/* reference.cpp:77-91 (broadcast when b has one row) */
int hvo_xor_bind(const uint8_t* a, size_t a_rows, const uint8_t* b, size_t b_rows, size_t dim,
                 uint8_t* out) {
  if (b_rows != a_rows && b_rows != 1) return HVO_INVALID_ARGUMENT;
  const int bc = b_rows == 1;
  for (size_t r = 0; r < a_rows; ++r) {
    for (size_t j = 0; j < dim; ++j) out[r * dim + j] = a[r * dim + j] ^ b[(bc ? 0 : r) * dim + j];
  }
  return HVO_OK;
}

/* reference.cpp:93-104: out bit (j + s) mod d = in bit j */
void hvo_rotate(const uint8_t* m, size_t rows, size_t dim, size_t shift, uint8_t* out) {
  if (dim == 0) return;
  const size_t s = shift % dim;
  for (size_t r = 0; r < rows; ++r) {
    for (size_t j = 0; j < dim; ++j) out[r * dim + (j + s) % dim] = m[r * dim + j];
  }
}

/* reference.cpp:106-114 */
void hvo_horizontal_sum(const uint8_t* m, size_t rows, size_t dim, uint64_t* out) {
  for (size_t r = 0; r < rows; ++r) {
    uint64_t s = 0;
    for (size_t j = 0; j < dim; ++j) s += m[r * dim + j];
    out[r] = s;
  }
}

/* reference.cpp:116-124 */
void hvo_transpose(const uint8_t* m, size_t rows, size_t dim, uint8_t* out) {
  for (size_t r = 0; r < rows; ++r) {
    for (size_t j = 0; j < dim; ++j) out[j * rows + r] = m[r * dim + j];
  }
}

/* reference.cpp:126-134 */
void hvo_vertical_sum(const uint8_t* m, size_t rows, size_t dim, uint64_t* out) {
  for (size_t j = 0; j < dim; ++j) out[j] = 0;
  for (size_t r = 0; r < rows; ++r) {
    for (size_t j = 0; j < dim; ++j) out[j] += m[r * dim + j];
  }
}

/* reference.cpp:136-155 (2c > n -> 1, 2c < n -> 0, else tiebreak) */
long long hvo_majority_binarize(const uint64_t* counts, size_t dim, uint64_t n,
                                const uint8_t* tiebreak, uint8_t* out) {
  for (size_t j = 0; j < dim; ++j) {
    if (counts[j] > n) return (long long)j;
    const uint64_t twice = 2 * counts[j];
    out[j] = twice > n ? 1 : (twice < n ? 0 : tiebreak[j]);
  }
  return -1;
}

/* ======================================================================= */
/* Discretizer (encoding.cpp:93-154)                                       */
/* ======================================================================= */

/* encoding.cpp:93-119: first-row init, strict < / > updates */
int hvo_fit_discretizer(const double* data, size_t rows, size_t features, size_t bins,
                        double* min_out, double* max_out) {
  if (rows == 0 || features == 0) return HVO_INVALID_ARGUMENT;
  if (bins < 2) return HVO_INVALID_ARGUMENT;
  for (size_t f = 0; f < features; ++f) min_out[f] = max_out[f] = data[f];
  for (size_t r = 1; r < rows; ++r) {
    for (size_t f = 0; f < features; ++f) {
      const double v = data[r * features + f];
      if (v < min_out[f]) min_out[f] = v;
      if (v > max_out[f]) max_out[f] = v;
    }
  }
  return HVO_OK;
}

/* encoding.cpp:121-139 (per value) and :141-154 (row-wise) */
void hvo_discretize_matrix(const double* data, size_t rows, size_t features, const double* mn,
                           const double* mx, size_t bins, uint32_t* out) {
  for (size_t r = 0; r < rows; ++r) {
    for (size_t f = 0; f < features; ++f) {
      uint32_t b = 0;
      if (!(mn[f] == mx[f])) {
        const double t = floor((data[r * features + f] - mn[f]) / (mx[f] - mn[f]) * (double)bins);
        const double top = (double)(bins - 1);
        if (t >= top) b = (uint32_t)(bins - 1);
        else if (t > 0.0) b = (uint32_t)t;
      }
      out[r * features + f] = b;
    }
  }
}

/* ======================================================================= */
/* Encode (reference.cpp:202-267; bin checks as encoding.cpp:43-55)        */
/* ======================================================================= */

int hvo_encode_batch(const uint32_t* bin_rows, size_t rows, size_t features,
                     const uint8_t* id_dense, const uint8_t* value_dense, size_t bins,
                     size_t dim, int binding, const uint8_t* tiebreak, uint8_t* out,
                     long long* bad_index) {
  if (bad_index) *bad_index = -1;
  if (features == 0 || dim == 0) return HVO_INVALID_ARGUMENT;
  uint64_t* counts = (uint64_t*)malloc(dim * sizeof(uint64_t));
  int status = HVO_OK;
  for (size_t r = 0; r < rows && status == HVO_OK; ++r) {
    const uint32_t* b = bin_rows + r * features;
    for (size_t f = 0; f < features; ++f) {
      if (b[f] >= bins) { /* encoding.cpp:48-54 */
        if (bad_index) *bad_index = (long long)(r * features + f);
        status = HVO_INVALID_ARGUMENT;
        break;
      }
    }
    if (status != HVO_OK) break;
    uint8_t* o = out + r * dim;
    switch (binding) {
      case HVO_BIND_ID_LEVEL: /* reference.cpp:217-226 */
        for (size_t j = 0; j < dim; ++j) counts[j] = 0;
        for (size_t f = 0; f < features; ++f) {
          for (size_t j = 0; j < dim; ++j) counts[j] += id_dense[f * dim + j] ^ value_dense[b[f] * dim + j];
        }
        hvo_majority_binarize(counts, dim, features, tiebreak, o);
        break;
      case HVO_BIND_PERMUTATION: /* reference.cpp:227-237 */
        for (size_t j = 0; j < dim; ++j) counts[j] = 0;
        for (size_t f = 0; f < features; ++f) {
          for (size_t j = 0; j < dim; ++j) counts[j] += value_dense[b[f] * dim + (j + dim - (f % dim)) % dim];
        }
        hvo_majority_binarize(counts, dim, features, tiebreak, o);
        break;
      case HVO_BIND_APPENDING: { /* reference.cpp:238-249 */
        const size_t seg = dim / features;
        if (seg == 0) { status = HVO_INVALID_ARGUMENT; break; }
        memset(o, 0, dim);
        for (size_t f = 0; f < features; ++f) {
          for (size_t j = 0; j < seg; ++j) o[f * seg + j] = value_dense[b[f] * dim + j];
        }
        break;
      }
      default: status = HVO_INVALID_ARGUMENT;
    }
  }
  free(counts);
  return status;
}

/* ======================================================================= */
/* Model (reference.cpp:21-73, 269-388)                                   */
/* ======================================================================= */

/* reference.cpp:269-282 */
void hvo_refresh_binarization(hvo_model* m, size_t c) {
  const size_t d = m->dim;
  const double total = m->class_weight[c];
  for (size_t j = 0; j < d; ++j) {
    const double twice = 2.0 * m->accumulators[c * d + j];
    uint8_t bit;
    if (twice > total) bit = 1;
    else if (twice < total) bit = 0;
    else bit = m->tiebreak[j];
    m->class_vectors[c * d + j] = bit;
  }
}

/* reference.cpp:21-55 */
static int class_scores(const hvo_model* m, const uint8_t* cv, const double* acc,
                        const uint8_t* row, double* scores) {
  const size_t cc = m->class_count, d = m->dim;
  if (m->metric == HVO_METRIC_HAMMING) {
    for (size_t c = 0; c < cc; ++c) {
      uint64_t diff = 0;
      for (size_t j = 0; j < d; ++j) diff += cv[c * d + j] != row[j];
      scores[c] = (double)diff / (double)d;
    }
    return HVO_OK;
  }
  for (size_t c = 0; c < cc; ++c) {
    double dot = 0.0, an = 0.0, rn = 0.0;
    for (size_t j = 0; j < d; ++j) {
      const double a = acc[c * d + j];
      const double b = (double)row[j];
      dot += a * b;
      an += a * a;
      rn += b * b;
    }
    if (rn == 0.0) return HVO_DOMAIN_ERROR;
    scores[c] = an == 0.0 ? -INFINITY : dot / (sqrt(an) * sqrt(rn));
  }
  return HVO_OK;
}

/* reference.cpp:57-65: strict comparison, lowest index wins ties */
static size_t pick_label(int metric, const double* s, size_t n) {
  size_t best = 0;
  for (size_t c = 1; c < n; ++c) {
    const int better = metric == HVO_METRIC_HAMMING ? s[c] < s[best] : s[c] > s[best];
    if (better) best = c;
  }
  return best;
}

/* reference.cpp:69-73 */
static double score_to_delta(int metric, double score) {
  if (metric == HVO_METRIC_HAMMING) return score;
  if (isinf(score)) return 1.0;
  return (1.0 - score) / 2.0;
}

/* reference.cpp:292-317 */
int hvo_train_classical(hvo_model* m, const uint8_t* encoded, size_t rows, const int32_t* labels) {
  const size_t cc = m->class_count, d = m->dim;
  for (size_t i = 0; i < cc * d; ++i) m->accumulators[i] = 0.0;
  for (size_t c = 0; c < cc; ++c) { m->class_weight[c] = 0.0; m->sample_counts[c] = 0; }
  for (size_t i = 0; i < rows; ++i) {
    const int32_t y = labels[i];
    if (y < 0 || (size_t)y >= cc) return HVO_INVALID_ARGUMENT;
    for (size_t j = 0; j < d; ++j) m->accumulators[(size_t)y * d + j] += (double)encoded[i * d + j];
    m->class_weight[y] += 1.0;
    m->sample_counts[y] += 1;
  }
  for (size_t c = 0; c < cc; ++c) hvo_refresh_binarization(m, c);
  return HVO_OK;
}

/* reference.cpp:319-351 */
int hvo_online_update(hvo_model* m, const uint8_t* batch, size_t rows, const int32_t* labels,
                      const uint8_t* snap_cv, const double* snap_acc) {
  const size_t cc = m->class_count, d = m->dim;
  double* scores = (double*)malloc(cc * sizeof(double));
  uint8_t* touched = (uint8_t*)calloc(cc, 1);
  int status = HVO_OK;
  for (size_t i = 0; i < rows; ++i) {
    const int32_t y = labels[i];
    if (y < 0 || (size_t)y >= cc) { status = HVO_INVALID_ARGUMENT; break; }
    const size_t truth = (size_t)y;
    status = class_scores(m, snap_cv, snap_acc, batch + i * d, scores);
    if (status != HVO_OK) break;
    const size_t pred = pick_label(m->metric, scores, cc);
    const double dt = score_to_delta(m->metric, scores[truth]);
    for (size_t j = 0; j < d; ++j) m->accumulators[truth * d + j] += dt * (double)batch[i * d + j];
    m->class_weight[truth] += dt;
    m->sample_counts[truth] += 1;
    touched[truth] = 1;
    if (pred != truth) {
      const double dw = score_to_delta(m->metric, scores[pred]);
      const double penalty = m->gamma * (1.0 - dw);
      for (size_t j = 0; j < d; ++j) m->accumulators[pred * d + j] -= penalty * (double)batch[i * d + j];
      touched[pred] = 1;
    }
  }
  for (size_t c = 0; c < cc; ++c) {
    if (touched[c]) hvo_refresh_binarization(m, c);
  }
  free(scores);
  free(touched);
  return status;
}

/* reference.cpp:353-376 (bootstrap on the first batch, then every batch
 * including the first gets an online pass against its start snapshot) */
int hvo_train_online(hvo_model* m, const uint8_t* encoded, size_t rows, const int32_t* labels,
                     size_t batch_size) {
  if (batch_size == 0) return HVO_INVALID_ARGUMENT;
  const size_t cc = m->class_count, d = m->dim;
  const size_t first = batch_size < rows ? batch_size : rows;
  int status = hvo_train_classical(m, encoded, first, labels);
  if (status != HVO_OK) return status;
  uint8_t* snap_cv = (uint8_t*)malloc(cc * d);
  double* snap_acc = (double*)malloc(cc * d * sizeof(double));
  for (size_t start = 0; start < rows && status == HVO_OK; start += batch_size) {
    const size_t end = start + batch_size < rows ? start + batch_size : rows;
    memcpy(snap_cv, m->class_vectors, cc * d);
    memcpy(snap_acc, m->accumulators, cc * d * sizeof(double));
    status = hvo_online_update(m, encoded + start * d, end - start, labels + start, snap_cv, snap_acc);
  }
  free(snap_cv);
  free(snap_acc);
  return status;
}

/* reference.cpp:378-388 */
int hvo_predict(const hvo_model* m, const uint8_t* encoded, size_t rows, int32_t* labels,
                double* distances) {
  const size_t cc = m->class_count, d = m->dim;
  double* scores = (double*)malloc(cc * sizeof(double));
  int status = HVO_OK;
  for (size_t i = 0; i < rows; ++i) {
    status = class_scores(m, m->class_vectors, m->accumulators, encoded + i * d, scores);
    if (status != HVO_OK) break;
    labels[i] = (int32_t)pick_label(m->metric, scores, cc);
    if (distances) memcpy(distances + i * cc, scores, cc * sizeof(double));
  }
  free(scores);
  return status;
}

/* ======================================================================= */
/* Bench workload generator (include/hvb200_synth.h), exposed so tests can  */
/* pin the Python restatement and the device generator against it.         */
/* ======================================================================= */
#include "../include/hvb200_synth.h"

void hvo_synth(uint64_t row0, size_t rows, size_t features, size_t classes, size_t bins, int kind,
               uint64_t seed, uint32_t* bins_out, int32_t* labels_out) {
  for (size_t r = 0; r < rows; ++r) {
    const int32_t y = hvs_label(row0 + r, (uint32_t)classes, kind);
    labels_out[r] = y;
    for (size_t f = 0; f < features; ++f) {
      bins_out[r * features + f] = hvs_bin(row0 + r, (uint32_t)f, (uint32_t)features, y, (uint32_t)bins, seed);
    }
  }
}

/* ======================================================================= */
/* Reference test-support generator synth::make_synth                      */
/* (tests/support/synth.cpp:9-47, defaults synth.hpp:14-22): class i % C,   */
/* feature value = centre of bin centre_bin(c, f) + uniform jitter from one */
/* mt19937_64 next_unit() per (row, feature) in row-major order.            */
/* ======================================================================= */

/* synth.cpp:9-14 */
static size_t synth_centre_bin(size_t cls, size_t feature, size_t grid_bins) {
  return (cls * (feature + 1) + 3 * feature) % grid_bins;
}

/* synth.cpp:16-47 (segments = 1: no segment column) */
int hvo_make_synth(size_t rows, size_t features, size_t classes, size_t grid_bins, double jitter, uint64_t seed,
                   double* X, int32_t* y) {
  if (rows == 0 || features == 0 || classes == 0 || grid_bins == 0) return HVO_INVALID_ARGUMENT;
  hvo_rng* rng = (hvo_rng*)malloc(sizeof(hvo_rng));
  hvo_rng_seed(rng, seed);
  const double width = 1.0 / (double)grid_bins;
  for (size_t i = 0; i < rows; ++i) {
    const size_t cls = i % classes;
    y[i] = (int32_t)cls;
    for (size_t f = 0; f < features; ++f) {
      const double centre = ((double)synth_centre_bin(cls, f, grid_bins) + 0.5) * width;
      const double noise = jitter * (2.0 * hvo_rng_next_unit(rng) - 1.0) * 0.5 * width;
      X[i * features + f] = centre + noise;
    }
  }
  free(rng);
  return HVO_OK;
}

/* ======================================================================= */
/* Evaluation (eval.cpp:12-116)                                            */
/* ======================================================================= */

/* eval.cpp:12-37: centred majority over `window` in-bounds samples, the
 * window shifted inward at the edges, ties -> 1. Validation (window odd and
 * >= 1, labels 0/1) happens before the empty / window-1 early return. */
int hvo_smooth_labels(const int32_t* labels, size_t n, size_t window, int32_t* out, uint64_t* bad) {
  if (window == 0 || window % 2 == 0) {
    *bad = window;
    return HVO_INVALID_ARGUMENT;
  }
  for (size_t i = 0; i < n; ++i) {
    if (labels[i] != 0 && labels[i] != 1) {
      *bad = i;
      return HVO_INVALID_ARGUMENT;
    }
  }
  if (n == 0) return HVO_OK;
  if (window == 1) {
    memcpy(out, labels, n * sizeof(int32_t));
    return HVO_OK;
  }
  const size_t len = window < n ? window : n;
  const size_t half = (window - 1) / 2;
  size_t* prefix = (size_t*)calloc(n + 1, sizeof(size_t));
  for (size_t i = 0; i < n; ++i) prefix[i + 1] = prefix[i] + (size_t)labels[i];
  for (size_t i = 0; i < n; ++i) {
    size_t start = i > half ? i - half : 0;
    if (start > n - len) start = n - len;
    const size_t ones = prefix[start + len] - prefix[start];
    out[i] = 2 * ones >= len ? 1 : 0;
  }
  free(prefix);
  return HVO_OK;
}

/* eval.cpp:39-77: confusion against one positive class; accuracy over exact
 * matches; a ratio with a zero denominator stays absent (NaN here). */
int hvo_sample_metrics(const int32_t* pred, size_t n_pred, const int32_t* truth, size_t n_truth,
                       int positive_class, uint64_t* counts, double* ratios) {
  if (n_pred != n_truth || n_pred == 0) return HVO_INVALID_ARGUMENT;
  uint64_t tp = 0, fp = 0, tn = 0, fn = 0, exact = 0;
  for (size_t i = 0; i < n_pred; ++i) {
    if (pred[i] == truth[i]) ++exact;
    const int p = pred[i] == positive_class, t = truth[i] == positive_class;
    if (p && t) ++tp;
    else if (p) ++fp;
    else if (t) ++fn;
    else ++tn;
  }
  counts[0] = tp; counts[1] = fp; counts[2] = tn; counts[3] = fn; counts[4] = exact;
  ratios[0] = (double)exact / (double)n_pred;
  ratios[1] = tp + fn > 0 ? (double)tp / (double)(tp + fn) : NAN;
  ratios[2] = tp + fp > 0 ? (double)tp / (double)(tp + fp) : NAN;
  ratios[3] = NAN;
  if (!isnan(ratios[1]) && !isnan(ratios[2]) && ratios[1] + ratios[2] > 0.0) {
    ratios[3] = 2.0 * ratios[2] * ratios[1] / (ratios[2] + ratios[1]);
  }
  return HVO_OK;
}

/* eval.cpp:79-116: truth episodes (maximal positive-truth runs) detected iff a
 * sample in the run is predicted positive; false-positive episodes are
 * maximal positive-prediction runs with no positive truth inside. */
int hvo_episode_metrics(const int32_t* pred, size_t n_pred, const int32_t* truth, size_t n_truth,
                        int positive_class, uint64_t* out) {
  if (n_pred != n_truth) return HVO_INVALID_ARGUMENT;
  const size_t n = n_pred;
  uint64_t detected = 0, total = 0, fpe = 0;
  for (size_t i = 0; i < n;) {
    if (truth[i] != positive_class) { ++i; continue; }
    int hit = 0;
    while (i < n && truth[i] == positive_class) { hit = hit || pred[i] == positive_class; ++i; }
    ++total;
    if (hit) ++detected;
  }
  for (size_t i = 0; i < n;) {
    if (pred[i] != positive_class) { ++i; continue; }
    int overlaps = 0;
    while (i < n && pred[i] == positive_class) { overlaps = overlaps || truth[i] == positive_class; ++i; }
    if (!overlaps) ++fpe;
  }
  out[0] = detected; out[1] = total; out[2] = fpe;
  return HVO_OK;
}
