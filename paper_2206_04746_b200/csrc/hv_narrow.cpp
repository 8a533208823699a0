// hv_narrow.cpp — the host narrowing kernel of the staging pipeline
// (hv_stage.cu): uint32 bin rows (the reference API type, encoding.hpp:85-93)
// -> uint8 rows of pitch ldb with zero padding, returning the largest bin seen
// so the caller validates against B with one compare per piece
// (encoding.cpp:43-55).
//
// Compiled by the host compiler (not nvcc) so the AVX-512 path can use
// intrinsics. That path is memory-bound on the host: per bin it reads 4 bytes
// and writes 1; the writes go to pinned staging that the GPU DMAs from, so
// they are non-temporal (no read-for-ownership of the destination lines, and
// nothing left in the cache the DMA engine would have to snoop).
#include <immintrin.h>

#include <cstddef>
#include <cstdint>

// declared in hv_stage.h (not included: it pulls in the CUDA headers)

namespace hvb {
namespace {

template <int kDummy>
inline uint32_t narrow_rows_impl(const uint32_t* __restrict__ in, size_t F, size_t r0, size_t r1,
                                 uint8_t* __restrict__ out, size_t ldb) {
  uint32_t mx = 0;
  for (size_t r = r0; r < r1; ++r) {
    const uint32_t* s = in + r * F;
    uint8_t* d = out + r * ldb;
    for (size_t f = 0; f < F; ++f) {
      const uint32_t v = s[f];
      mx = v > mx ? v : mx;
      d[f] = static_cast<uint8_t>(v);
    }
    for (size_t f = F; f < ldb; ++f) d[f] = 0;
  }
  return mx;
}

__attribute__((target("avx2"))) uint32_t narrow_rows_avx2(const uint32_t* in, size_t F, size_t r0, size_t r1,
                                                          uint8_t* out, size_t ldb) {
  return narrow_rows_impl<1>(in, F, r0, r1, out, ldb);
}

uint32_t narrow_rows_base(const uint32_t* in, size_t F, size_t r0, size_t r1, uint8_t* out, size_t ldb) {
  return narrow_rows_impl<0>(in, F, r0, r1, out, ldb);
}

// 16 bins per step: masked 64-byte load (zeros past F, which also writes the
// row padding), unsigned max, VPMOVDB truncation, 16-byte streaming store.
// Needs 16-byte aligned rows (out and ldb multiples of 16).
__attribute__((target("avx512f,avx512bw,avx512vl"))) uint32_t narrow_rows_avx512(const uint32_t* in, size_t F,
                                                                                 size_t r0, size_t r1, uint8_t* out,
                                                                                 size_t ldb) {
  __m512i mx = _mm512_setzero_si512();
  for (size_t r = r0; r < r1; ++r) {
    const uint32_t* s = in + r * F;
    uint8_t* d = out + r * ldb;
    size_t f = 0;
    for (; f + 16 <= F; f += 16) {
      const __m512i v = _mm512_loadu_si512(s + f);
      mx = _mm512_max_epu32(mx, v);
      _mm_stream_si128(reinterpret_cast<__m128i*>(d + f), _mm512_cvtepi32_epi8(v));
    }
    for (; f < ldb; f += 16) {
      const size_t left = f < F ? F - f : 0;
      const __mmask16 m = static_cast<__mmask16>((1u << left) - 1u);
      const __m512i v = _mm512_maskz_loadu_epi32(m, s + f);
      mx = _mm512_max_epu32(mx, v);
      _mm_stream_si128(reinterpret_cast<__m128i*>(d + f), _mm512_cvtepi32_epi8(v));
    }
  }
  _mm_sfence();  // the streaming stores are visible before the piece is reported done
  return _mm512_reduce_max_epu32(mx);
}

}  // namespace

uint32_t narrow_rows(const uint32_t* in, size_t F, size_t r0, size_t r1, uint8_t* out, size_t ldb) {
  static const int level = __builtin_cpu_supports("avx512bw") && __builtin_cpu_supports("avx512vl") ? 2
                           : __builtin_cpu_supports("avx2")                                          ? 1
                                                                                                      : 0;
  const bool aligned16 = ((reinterpret_cast<uintptr_t>(out) | ldb) & 15u) == 0;
  if (level == 2 && aligned16 && ldb >= F) return narrow_rows_avx512(in, F, r0, r1, out, ldb);
  if (level >= 1) return narrow_rows_avx2(in, F, r0, r1, out, ldb);
  return narrow_rows_base(in, F, r0, r1, out, ldb);
}

}  // namespace hvb
