// hv_internal.cuh — shared plumbing for libhvb200 (context, errors, device
// scratch, launch accounting) and the bit-sliced counting primitives used by
// every counting kernel.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <utility>

#include "hvb200.h"

namespace hvb {

// --------------------------------------------------------------- errors ----
struct Error {
  hv_status status;
  std::string message;
};

[[noreturn]] inline void fail(hv_status s, std::string msg) { throw Error{s, std::move(msg)}; }
[[noreturn]] inline void invalid(std::string msg) { fail(HV_ERR_INVALID_ARGUMENT, std::move(msg)); }

void set_last_error(const std::string& msg);

template <class F>
hv_status guarded(F&& f) {
  try {
    f();
    return HV_OK;
  } catch (const Error& e) {
    set_last_error(e.message);
    return e.status;
  } catch (const std::bad_alloc&) {
    set_last_error("out of host memory");
    return HV_ERR_RUNTIME;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return HV_ERR_RUNTIME;
  }
}

inline void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    fail(HV_ERR_CUDA, std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")");
  }
}

// Every kernel launch goes through this counter (bench.py reports it as
// gpu_launches; tests assert the CUDA path actually ran).
extern std::atomic<uint64_t> g_launches;
inline void launched(const char* what) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  ck(cudaPeekAtLastError(), what);
}

// ------------------------------------------------------ latched errors ----
// Data-dependent failures found inside kernels: the minimum offending flat
// index per kind is recorded with atomicMin; UINT64_MAX = none.
enum ErrKind { kErrBin = 0, kErrLabel = 1, kErrByte = 2, kErrCount = 3, kErrZeroQuery = 4, kErrKinds = 5 };

__device__ __forceinline__ void latch(unsigned long long* err, int kind, unsigned long long index) {
  atomicMin(err + kind, index);
}

struct HostStager;

}  // namespace hvb

struct hv_context {
  int device = 0;
  cudaStream_t own = nullptr;
  cudaStream_t stream = nullptr;
  cudaStream_t aux = nullptr;           // second stream for copy/compute overlap
  unsigned long long* d_err = nullptr;  // hvb::kErrKinds slots
  int sm_count = 148;
  size_t smem_optin = 0;
  static constexpr unsigned kCounters = 64;
  unsigned int* d_counters = nullptr;   // dynamic-scheduling counters (ring)
  unsigned next_counter = 0;
  hvb::HostStager* stager = nullptr;    // host narrowing pool + pinned slots (lazy)
};

namespace hvb {

hv_context* require(hv_context* ctx);

// Reads and resets the latch; returns the slots.
void read_latch(hv_context* ctx, unsigned long long out[kErrKinds]);
void reset_latch(hv_context* ctx);

// Stream-ordered device allocation (cudaMallocAsync pool), freed on scope exit.
template <class T>
struct DevBuf {
  T* ptr = nullptr;
  size_t n = 0;
  cudaStream_t stream = nullptr;
  DevBuf() = default;
  DevBuf(size_t count, cudaStream_t s) : n(count), stream(s) {
    if (count) ck(cudaMallocAsync(reinterpret_cast<void**>(&ptr), count * sizeof(T), s), "cudaMallocAsync");
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : ptr(o.ptr), n(o.n), stream(o.stream) { o.ptr = nullptr; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      if (ptr) cudaFreeAsync(ptr, stream);
      ptr = o.ptr;
      n = o.n;
      stream = o.stream;
      o.ptr = nullptr;
    }
    return *this;
  }
  ~DevBuf() {
    if (ptr) cudaFreeAsync(ptr, stream);
  }
  size_t bytes() const { return n * sizeof(T); }
  void upload(const T* host) {
    if (n) ck(cudaMemcpyAsync(ptr, host, bytes(), cudaMemcpyHostToDevice, stream), "H2D");
  }
  void download(T* host) const {
    if (n) ck(cudaMemcpyAsync(host, ptr, bytes(), cudaMemcpyDeviceToHost, stream), "D2H");
  }
  void zero() {
    if (n) ck(cudaMemsetAsync(ptr, 0, bytes(), stream), "memset");
  }
};

inline void sync(hv_context* ctx) { ck(cudaStreamSynchronize(ctx->stream), "cudaStreamSynchronize"); }

inline size_t words_per_row(size_t dim) { return (dim + 31) / 32; }
inline uint32_t pad_mask_host(size_t dim) {
  const size_t rem = dim % 32;
  return rem == 0 ? ~0u : ((1u << rem) - 1u);  // valid-bit mask of the last word
}
inline unsigned grid_for(size_t n, unsigned block, unsigned cap = 1u << 30) {
  size_t g = (n + block - 1) / block;
  if (g == 0) g = 1;
  if (g > cap) g = cap;
  return static_cast<unsigned>(g);
}

// Column counts over a permuted, class-segmented row sequence (hv_bits.cu).
// ldm: row pitch in words (0 = W); pitched 16-byte-aligned rows (ldm % 4 == 0)
// take the TMA-staged kernel.
void launch_column_count_u32(cudaStream_t st, const uint32_t* m, uint32_t W, const uint32_t* perm,
                             const uint64_t* seg_off, uint32_t nseg, uint64_t max_pos, uint32_t* counts,
                             uint32_t ldm = 0);
// Label bucketing for class counts (hv_model.cu): histogram (validated, into
// a zeroed hist), segment offsets, class-sorted permutation; class_rows += hist.
void label_bucket_device(hv_context* ctx, cudaStream_t st, const int32_t* labels, size_t rows, size_t C,
                         uint32_t* hist, uint64_t* offsets, uint32_t* cursor, uint32_t* perm,
                         uint64_t* class_rows = nullptr);
// Same, flushing into `single`, or (dsts_dev != nullptr) into the ndst count
// buffers listed in the device array dsts_dev (every rank's, over peer memory).
void launch_column_count_peers(cudaStream_t st, const uint32_t* m, uint32_t W, const uint32_t* perm,
                               const uint64_t* seg_off, uint32_t nseg, uint64_t max_pos, uint32_t* single,
                               uint32_t* const* dsts_dev, uint32_t ndst, uint32_t ldm = 0);

// Encoder entry points shared with the fold pipeline (hv_encode.cu). Words
// [w0, w0 + wcount) of every row are written to out[row * ldo + k]; wcount = 0
// means the whole row (w0 = 0, wcount = ldo = W).
void encode_device(hv_context* ctx, cudaStream_t st, const uint8_t* bins8, size_t ldb, size_t rows, size_t F,
                   const uint32_t* id, const uint32_t* val, size_t B, size_t D, hv_binding binding,
                   const uint32_t* tie, uint32_t* out, bool allow_fast = true, size_t w0 = 0, size_t wcount = 0,
                   size_t ldo = 0);
void narrow_device(hv_context* ctx, cudaStream_t st, const uint32_t* bins32, size_t rows, size_t F, size_t B,
                   uint8_t* bins8, size_t ldb, uint64_t flat_base);
inline size_t bins_pitch(size_t F) { return (F + 63) / 64 * 64; }
// Device bins are one byte each: the reference accepts any bin count >= 2
// (encoding.cpp:43-55), the device path up to 256 and rejects more, loudly,
// rather than truncating bins into neighbouring bytes.
inline void check_bins_u8(size_t B, const char* fn) {
  if (B > 256) {
    invalid(std::string(fn) + ": bins = " + std::to_string(B) + " exceeds 256, the device encoder's uint8 bin range");
  }
}
// Discretizer on HBM-resident fp64 features over rows idx[0..n) (idx may be
// null: rows 0..n): fit (encoding.cpp:93-119) and discretize to uint8 bins.
void fit_discretizer_device(hv_context* ctx, cudaStream_t st, const double* X, size_t F, const uint64_t* idx,
                            size_t n, double* mn, double* mx);
void discretize_rows_device(hv_context* ctx, cudaStream_t st, const double* X, size_t F, const uint64_t* idx,
                            size_t n, const double* mn, const double* mx, size_t B, uint8_t* out, size_t ldb);
// Tensor-core ID-level encoder (hv_encode_tc.cu): whole rows, B <= 16; false
// when the shape is not supported (nothing launched).
bool launch_tc(hv_context* ctx, cudaStream_t st, const uint8_t* bins8, uint32_t ldb, uint64_t rows, uint32_t F,
               const uint32_t* id, const uint32_t* val, uint32_t B, uint32_t D, uint32_t W, const uint32_t* tie,
               uint32_t* out, uint32_t ldo);
bool launch_tt(hv_context* ctx, cudaStream_t st, const uint8_t* bins8, uint32_t ldb, uint64_t rows, uint32_t F,
               const uint32_t* id, const uint32_t* val, uint32_t B, uint32_t D, uint32_t W, const uint32_t* tie,
               uint32_t* out, uint32_t w0, uint32_t wcount, uint32_t ldo, bool perm = false,
               const unsigned long long* ready = nullptr);

// Online training, Hamming metric: every batch in one persistent cooperative
// kernel (hv_online.cu); acc/weight/counts/cv hold the bootstrap state.
// tcgen05 many-class scan (hv_predict_tc.cu): fills best[] (argmin keys, pre-set
// to ~0) and the optional dist / pops; false when enc is not 16-byte aligned.
bool predict_tc_launch(hv_context* ctx, cudaStream_t st, const uint32_t* cv, size_t C, size_t D, const uint32_t* enc,
                       size_t rows, const uint32_t* cpop, unsigned long long* best, double* dist, uint32_t* pops);
// rows x C Hamming popcounts on the tensor cores, split over K to fill the GPU
// (online scoring): ADDS into pops, which must be zero; img:
// tc_image_bytes(C, D) bytes, cpop: C words of scratch; requires tc_usable(enc, D)
size_t tc_image_bytes(size_t C, size_t D);
bool tc_usable(const uint32_t* enc, size_t D);
void popc_tc_split(hv_context* ctx, cudaStream_t st, const uint32_t* cv, size_t C, size_t D, const uint32_t* enc,
                   size_t rows, uint32_t* cpop, uint32_t* pops, uint8_t* img);
void train_online_persistent(hv_context* ctx, cudaStream_t st, const uint32_t* enc, size_t rows, size_t D,
                             const int32_t* labels, size_t C, size_t bsz, double gamma, const uint32_t* tie,
                             double* acc, double* weight, uint64_t* counts, uint32_t* cv);

// Host-side codebook helpers shared by several entry points (hv_host.cpp).
// hv_eval.cu — eval.cpp:12-116 on device labels
void smooth_labels_device(hv_context* ctx, cudaStream_t st, const int32_t* labels, size_t n, size_t window,
                          int32_t* out);
void confusion_device(hv_context* ctx, cudaStream_t st, const int32_t* pred, const int32_t* truth, size_t n,
                      int positive, unsigned long long* out5);
void episodes_device(hv_context* ctx, cudaStream_t st, const int32_t* pred, const int32_t* truth, size_t n,
                     int positive, unsigned long long* out3);
void fill_report(const unsigned long long c5[5], const unsigned long long e3[3], size_t n, hv_eval_report* r);
void scatter_labels_device(hv_context* ctx, cudaStream_t st, const uint64_t* idx, size_t n, const int32_t* lab,
                           int32_t* predicted);
template <class T>
struct DevBuf;
size_t compact_tested_device(hv_context* ctx, cudaStream_t st, const int32_t* predicted, const int32_t* y,
                             size_t rows, DevBuf<uint64_t>& tested, DevBuf<int32_t>& pred_seq,
                             DevBuf<int32_t>& truth_seq);

void generate_random_words(size_t count, size_t dim, uint64_t seed, uint32_t* out);
uint64_t derive_seed(uint64_t seed, uint64_t tag);

// ----------------------------------------------------- device helpers ----
// Valid-bit mask of word w of a dim-bit row.
__device__ __forceinline__ uint32_t valid_mask(uint32_t w, uint32_t dim) {
  const uint32_t base = w * 32u;
  if (base + 32u <= dim) return 0xFFFFFFFFu;
  if (base >= dim) return 0u;
  return (1u << (dim - base)) - 1u;
}

// 32 bits starting at bit position `pos` of a packed row (zero past the row end).
__device__ __forceinline__ uint32_t get_bits32(const uint32_t* row, uint32_t words, uint64_t pos) {
  const uint32_t wi = static_cast<uint32_t>(pos >> 5);
  const uint32_t off = static_cast<uint32_t>(pos & 31u);
  const uint32_t lo = wi < words ? row[wi] : 0u;
  const uint32_t hi = wi + 1 < words ? row[wi + 1] : 0u;
  return __funnelshift_r(lo, hi, off);
}

// 32 bits starting at position p (0 <= p < dim) taken cyclically modulo dim:
// bit t of the result = row bit (p + t) mod dim for t < min(32, dim). Bits at
// t >= dim (only possible when dim < 32) are garbage; callers mask padding.
__device__ __forceinline__ uint32_t get_bits_cyclic(const uint32_t* row, uint32_t words, uint32_t dim,
                                                    uint32_t p) {
  const uint32_t first = dim - p;  // bits available before wrapping
  const uint32_t v = get_bits32(row, words, p);
  if (first >= 32u) return v;
  return (v & ((1u << first) - 1u)) | (get_bits32(row, words, 0) << first);
}

// Carry-save adder on bit-sliced words: a + b + c = l + 2h (per bit).
__device__ __forceinline__ void csa(uint32_t& h, uint32_t& l, uint32_t a, uint32_t b, uint32_t c) {
  const uint32_t u = a ^ b;
  h = (a & b) | (u & c);
  l = u ^ c;
}

// Harley–Seal bit-sliced counter: count = ones + 2 twos + 4 fours + 8 eights + 16 * hi.
template <int NH>
struct HSCounter {
  uint32_t ones = 0, twos = 0, fours = 0, eights = 0;
  uint32_t hi[NH];
  __device__ __forceinline__ HSCounter() {
#pragma unroll
    for (int k = 0; k < NH; ++k) hi[k] = 0;
  }
  // adds a weight-16 word into hi (ripple)
  __device__ __forceinline__ void add16w(uint32_t c) {
#pragma unroll
    for (int k = 0; k < NH; ++k) {
      const uint32_t t = hi[k] & c;
      hi[k] ^= c;
      c = t;
    }
  }
  // adds 16 input words
  __device__ __forceinline__ void add16(const uint32_t x[16]) {
    uint32_t twosA, twosB, foursA, foursB, eightsA, eightsB, sixteens;
    csa(twosA, ones, ones, x[0], x[1]);
    csa(twosB, ones, ones, x[2], x[3]);
    csa(foursA, twos, twos, twosA, twosB);
    csa(twosA, ones, ones, x[4], x[5]);
    csa(twosB, ones, ones, x[6], x[7]);
    csa(foursB, twos, twos, twosA, twosB);
    csa(eightsA, fours, fours, foursA, foursB);
    csa(twosA, ones, ones, x[8], x[9]);
    csa(twosB, ones, ones, x[10], x[11]);
    csa(foursA, twos, twos, twosA, twosB);
    csa(twosA, ones, ones, x[12], x[13]);
    csa(twosB, ones, ones, x[14], x[15]);
    csa(foursB, twos, twos, twosA, twosB);
    csa(eightsB, fours, fours, foursA, foursB);
    csa(sixteens, eights, eights, eightsA, eightsB);
    add16w(sixteens);
  }
  // adds 8 input words
  __device__ __forceinline__ void add8(const uint32_t x[8]) {
    uint32_t twosA, twosB, foursA, foursB, eightsA;
    csa(twosA, ones, ones, x[0], x[1]);
    csa(twosB, ones, ones, x[2], x[3]);
    csa(foursA, twos, twos, twosA, twosB);
    csa(twosA, ones, ones, x[4], x[5]);
    csa(twosB, ones, ones, x[6], x[7]);
    csa(foursB, twos, twos, twosA, twosB);
    csa(eightsA, fours, fours, foursA, foursB);
    const uint32_t sixteens = eights & eightsA;
    eights ^= eightsA;
    add16w(sixteens);
  }
  // plane k of the binary count (k < 4 + NH)
  __device__ __forceinline__ uint32_t plane(int k) const {
    switch (k) {
      case 0: return ones;
      case 1: return twos;
      case 2: return fours;
      case 3: return eights;
      default: return hi[k - 4];
    }
  }
  // per-bit count of bit position t
  __device__ __forceinline__ uint32_t count_of(int t) const {
    uint32_t c = ((ones >> t) & 1u) | (((twos >> t) & 1u) << 1) | (((fours >> t) & 1u) << 2) |
                 (((eights >> t) & 1u) << 3);
#pragma unroll
    for (int k = 0; k < NH; ++k) c |= ((hi[k] >> t) & 1u) << (4 + k);
    return c;
  }
  // Majority vote against a total n (kernels.cpp:142-160 / encoding.cpp:266-272):
  // bit = 2c > n ? 1 : 2c < n ? 0 : tie. Requires n < 2^(5+NH).
  __device__ __forceinline__ uint32_t majority(uint32_t n, uint32_t tie) const {
    const uint32_t half = n >> 1;
    uint32_t gt = 0u, eq = 0xFFFFFFFFu;
#pragma unroll
    for (int k = 3 + NH; k >= 0; --k) {
      const uint32_t p = plane(k);
      if ((half >> k) & 1u) {
        eq &= p;
      } else {
        gt |= eq & p;
        eq &= ~p;
      }
    }
    // c > half  <=> 2c > n (n odd: c >= half+1; n even: c > n/2)
    // c == half <=> 2c == n only when n is even; for odd n, 2c = n-1 < n -> 0.
    return gt | ((n & 1u) ? 0u : (eq & tie));
  }
};

// Number of high planes needed so that counts up to n fit: 16 * 2^NH > n.
inline int hs_high_planes(uint64_t n) {
  int nh = 1;
  while ((uint64_t(16) << nh) <= n) ++nh;
  return nh;
}

}  // namespace hvb
