// hv_host.cu — host side of libhvb200: error reporting, contexts, the
// reference-identical RNG / codebook generators and model bookkeeping.
//
// Codebooks are generated on the host with std::mt19937_64 exactly as the
// reference does (one engine draw per 32-bit word, rng.hpp:13-51,
// encoding.cpp:25-28, 156-255): they are a one-time, inherently sequential
// setup step (<1 ms per MB) and must be bit-identical, so there is nothing to
// gain from a device generator. They are uploaded once and stay resident.

#include <algorithm>
#include <cstdio>
#include <numeric>
#include <random>
#include <vector>

#include "hv_internal.cuh"
#include "hv_stage.h"

namespace hvb {

std::atomic<uint64_t> g_launches{0};

namespace {
thread_local std::string t_last_error;
}

void set_last_error(const std::string& msg) { t_last_error = msg; }

hv_context* require(hv_context* ctx) {
  if (ctx == nullptr) invalid("null hv_context");
  ck(cudaSetDevice(ctx->device), "cudaSetDevice");
  return ctx;
}

void reset_latch(hv_context* ctx) {
  ck(cudaMemsetAsync(ctx->d_err, 0xFF, sizeof(unsigned long long) * kErrKinds, ctx->stream), "latch reset");
}

void read_latch(hv_context* ctx, unsigned long long out[kErrKinds]) {
  ck(cudaMemcpyAsync(out, ctx->d_err, sizeof(unsigned long long) * kErrKinds, cudaMemcpyDeviceToHost,
                     ctx->stream),
     "latch read");
  sync(ctx);
}

// ---- rng.hpp:13-24 ----------------------------------------------------------
static uint64_t mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

uint64_t derive_seed(uint64_t seed, uint64_t tag) { return mix64(mix64(seed) ^ mix64(tag)); }

namespace {

struct Words {
  uint32_t* p;
  size_t rows, dim, wpr;
  uint32_t* row(size_t r) const { return p + r * wpr; }
  bool bit(size_t r, size_t j) const { return (row(r)[j >> 5] >> (j & 31)) & 1u; }
  void flip(size_t r, size_t j) const { row(r)[j >> 5] ^= 1u << (j & 31); }
  void put(size_t r, size_t j, bool v) const {
    const uint32_t m = 1u << (j & 31);
    uint32_t& w = row(r)[j >> 5];
    w = v ? (w | m) : (w & ~m);
  }
};

// One low-32-bit draw per word, then clear the padding bits of each row.
void fill_words(std::mt19937_64& eng, uint32_t* out, size_t rows, size_t dim) {
  const size_t wpr = words_per_row(dim);
  for (size_t i = 0; i < rows * wpr; ++i) out[i] = static_cast<uint32_t>(eng());
  if (dim % 32 && wpr) {
    const uint32_t keep = pad_mask_host(dim);
    for (size_t r = 0; r < rows; ++r) out[r * wpr + wpr - 1] &= keep;
  }
}

// Unbiased draw in [0, bound) by rejection (rng.hpp:37-42).
uint64_t draw_below(std::mt19937_64& eng, uint64_t bound) {
  const uint64_t floor = (0 - bound) % bound;
  uint64_t v = eng();
  while (v < floor) v = eng();
  return v % bound;
}

void copy_range(const Words& src, size_t sr, size_t soff, const Words& dst, size_t dr, size_t doff,
                size_t len) {
  for (size_t k = 0; k < len; ++k) dst.put(dr, doff + k, src.bit(sr, soff + k));
}

void scale_random(size_t bins, size_t dim, uint64_t seed, uint32_t* out) {
  if (bins < 2) invalid("generate_scale_random: need at least 2 bins");
  const size_t quota = dim / (2 * (bins - 1));
  if (quota == 0) {
    invalid("generate_scale_random: dim " + std::to_string(dim) + " too small for " + std::to_string(bins) +
            " bins (needs dim >= 2*(bins-1))");
  }
  const size_t wpr = words_per_row(dim);
  std::fill(out, out + bins * wpr, 0u);
  std::mt19937_64 eng(seed);
  fill_words(eng, out, 1, dim);
  // Each level flips `quota` never-flipped positions of the previous level,
  // drawn without replacement from the shrinking pool (partial Fisher-Yates).
  std::vector<size_t> pool(dim);
  std::iota(pool.begin(), pool.end(), size_t{0});
  size_t left = dim;
  Words m{out, bins, dim, wpr};
  for (size_t k = 1; k < bins; ++k) {
    std::copy(m.row(k - 1), m.row(k - 1) + wpr, m.row(k));
    for (size_t i = 0; i < quota; ++i) {
      const size_t pick = static_cast<size_t>(draw_below(eng, left));
      const size_t pos = pool[pick];
      pool[pick] = pool[--left];
      m.flip(k, pos);
    }
  }
}

void sandwich(size_t bins, size_t dim, uint64_t seed, uint32_t* out) {
  if (bins < 2) invalid("generate_sandwich: need at least 2 bins");
  if (dim % 2 != 0) invalid("generate_sandwich: dim must be even, got " + std::to_string(dim));
  const size_t wpr = words_per_row(dim);
  std::fill(out, out + bins * wpr, 0u);
  std::mt19937_64 eng(seed);
  Words m{out, bins, dim, wpr};
  for (size_t k = 0; k < bins; k += 2) fill_words(eng, m.row(k), 1, dim);
  const size_t half = dim / 2;
  std::vector<uint32_t> tail(words_per_row(half) + 1, 0u);
  Words t{tail.data(), 1, half, words_per_row(half)};
  for (size_t k = 1; k < bins; k += 2) {
    copy_range(m, k - 1, 0, m, k, 0, half);
    if (k + 1 < bins) {
      copy_range(m, k + 1, half, m, k, half, half);
    } else {
      fill_words(eng, tail.data(), 1, half);
      copy_range(t, 0, 0, m, k, half, half);
    }
  }
}

}  // namespace

void generate_random_words(size_t count, size_t dim, uint64_t seed, uint32_t* out) {
  std::mt19937_64 eng(seed);
  fill_words(eng, out, count, dim);
}

}  // namespace hvb

using namespace hvb;

extern "C" {

int hv_abi_version(void) { return HVB200_ABI_VERSION; }
const char* hv_last_error(void) { return hvb::t_last_error.c_str(); }
size_t hv_words_per_row(size_t dim) { return words_per_row(dim); }
uint64_t hv_kernel_launch_count(void) { return g_launches.load(); }

hv_status hv_context_create(int device, hv_context** out) {
  return guarded([&] {
    if (out == nullptr) invalid("hv_context_create: null output pointer");
    *out = nullptr;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
      cudaGetLastError();
      fail(HV_ERR_NO_DEVICE, "hv_context_create: no CUDA device available (libhvb200 has no CPU fallback)");
    }
    if (device < 0 || device >= n) invalid("hv_context_create: device " + std::to_string(device) + " out of range");
    cudaDeviceProp prop{};
    ck(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
    if (prop.major < 10) {
      fail(HV_ERR_NO_DEVICE, std::string("hv_context_create: ") + prop.name + " is sm_" +
                                 std::to_string(prop.major * 10 + prop.minor) +
                                 "; libhvb200 is built for sm_100a only");
    }
    ck(cudaSetDevice(device), "cudaSetDevice");
    auto* ctx = new hv_context();
    ctx->device = device;
    ctx->sm_count = prop.multiProcessorCount;
    ctx->smem_optin = prop.sharedMemPerBlockOptin;
    ck(cudaStreamCreateWithFlags(&ctx->own, cudaStreamNonBlocking), "cudaStreamCreate");
    ck(cudaStreamCreateWithFlags(&ctx->aux, cudaStreamNonBlocking), "cudaStreamCreate");
    ctx->stream = ctx->own;
    ck(cudaMalloc(&ctx->d_err, sizeof(unsigned long long) * kErrKinds), "cudaMalloc");
    ck(cudaMalloc(&ctx->d_counters, sizeof(unsigned int) * hv_context::kCounters), "cudaMalloc");
    // Keep freed scratch in the pool instead of returning it to the driver.
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    reset_latch(ctx);
    sync(ctx);
    *out = ctx;
  });
}

void hv_context_destroy(hv_context* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  cudaStreamSynchronize(ctx->aux);
  destroy_stager(ctx);
  cudaFree(ctx->d_err);
  cudaFree(ctx->d_counters);
  cudaStreamDestroy(ctx->aux);
  cudaStreamDestroy(ctx->own);
  delete ctx;
}

hv_status hv_context_set_stream(hv_context* ctx, void* stream) {
  return guarded([&] {
    require(ctx);
    ctx->stream = stream ? static_cast<cudaStream_t>(stream) : ctx->own;
  });
}

void* hv_context_stream(hv_context* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }

hv_status hv_context_synchronize(hv_context* ctx) {
  return guarded([&] { sync(require(ctx)); });
}

hv_status hv_dev_check(hv_context* ctx) {
  return guarded([&] {
    require(ctx);
    unsigned long long l[kErrKinds];
    read_latch(ctx, l);
    reset_latch(ctx);
    if (l[kErrBin] != ~0ull) invalid("encode: bin index out of range at flat index " + std::to_string(l[kErrBin]));
    if (l[kErrLabel] != ~0ull) invalid("label out of range at row " + std::to_string(l[kErrLabel]));
    if (l[kErrByte] != ~0ull) invalid("pack: non-binary entry at flat index " + std::to_string(l[kErrByte]));
    if (l[kErrCount] != ~0ull) invalid("majority_binarize: count exceeds total at position " + std::to_string(l[kErrCount]));
    if (l[kErrZeroQuery] != ~0ull) fail(HV_ERR_DOMAIN, "cosine_similarity: zero query vector");
  });
}

uint64_t hv_splitmix64(uint64_t x) { return mix64(x); }
uint64_t hv_derive_seed(uint64_t seed, uint64_t tag) { return derive_seed(seed, tag); }

hv_status hv_generate_random(size_t count, size_t dim, uint64_t seed, uint32_t* out) {
  return guarded([&] {
    if (count * words_per_row(dim) && !out) invalid("generate_random: null output");
    generate_random_words(count, dim, seed, out);
  });
}

hv_status hv_generate_scale_random(size_t bins, size_t dim, uint64_t seed, uint32_t* out) {
  return guarded([&] { scale_random(bins, dim, seed, out); });
}

hv_status hv_generate_sandwich(size_t bins, size_t dim, uint64_t seed, uint32_t* out) {
  return guarded([&] { sandwich(bins, dim, seed, out); });
}

// encoding.cpp:228-255: ID rows from derive_seed(seed, 1), Value rows from derive_seed(seed, 2)
hv_status hv_make_codebook(hv_generation generation, size_t features, size_t bins, size_t dim,
                           uint64_t seed, uint32_t* id_out, uint32_t* value_out) {
  return guarded([&] {
    if (features == 0 || dim == 0) invalid("make_codebook: features and dim must be >= 1");
    if (bins < 2) invalid("make_codebook: need at least 2 bins");
    generate_random_words(features, dim, derive_seed(seed, 1), id_out);
    const uint64_t vs = derive_seed(seed, 2);
    switch (generation) {
      case HV_GEN_RANDOM: generate_random_words(bins, dim, vs, value_out); break;
      case HV_GEN_SCALE_RANDOM: scale_random(bins, dim, vs, value_out); break;
      case HV_GEN_SANDWICH: sandwich(bins, dim, vs, value_out); break;
      default: fail(HV_ERR_LOGIC, "bad GenerationStrategy");
    }
  });
}

// model.cpp:178-181 (hamming_words / D in double)
double hv_hamming_distance_words(const uint32_t* a, const uint32_t* b, size_t dim) {
  const size_t w = words_per_row(dim);
  uint64_t diff = 0;
  for (size_t i = 0; i < w; ++i) diff += static_cast<uint64_t>(__builtin_popcount(a[i] ^ b[i]));
  return static_cast<double>(diff) / static_cast<double>(dim);
}

}  // extern "C"
