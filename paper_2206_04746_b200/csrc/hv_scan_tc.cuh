// hv_scan_tc.cuh — the many-class Hamming scan on the 5th-generation tensor
// cores (tcgen05, kind::i8, accumulators in TMEM).
//
//   popc(q ^ c) = |q| + |c| - 2 <q, c>
//
// CTA tile = 128 rows x 128 classes; the K dimension is the hypervector's bits,
// 256 per chunk (8 words). 256 threads: threads 2i and 2i+1 stage the two
// halves of row i and of class i — the packed words of the next chunk are loaded into
// registers while the current chunk's MMAs run, then every bit is spread to a
// byte (0/1, in a strided K order shared by both operands) and stored in the UMMA K-major no-swizzle layout (8-row x 16-byte core
// matrices: LBO = 128 B along K, SBO = 1024 B along M/N). One elected thread
// issues 4 tcgen05.mma (M=128, N=128, K=32 bytes each) per chunk and commits
// them to the stage's mbarrier; the other stage is being refilled meanwhile.
// The epilogue reads the s32 dot products out of TMEM (tcgen05.ld 32x32b:
// thread = row, so each row's argmin needs no shuffles).
#pragma once

#include <cstdint>

namespace hvb {
namespace tc {

constexpr int kM = 128, kN = 128;   // UMMA shape (rows x classes)
constexpr int kKBytes = 256;        // K bytes (= bits) per chunk: 8 words
constexpr int kStages = 2;
constexpr int kThreads = 256;  // 2 staging threads per row/class; warps 0-3 read TMEM
constexpr uint32_t kTileBytes = kM * kKBytes;  // 32 KB per operand and stage

struct __align__(1024) Smem {
  uint8_t a[kStages][kTileBytes];
  uint8_t b[kStages][kTileBytes];
  unsigned long long mbar[kStages];
  uint32_t tmem;
};
constexpr size_t kSmemBytes = sizeof(Smem) + 1024;  // + alignment slack

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// UMMA shared-memory descriptor, K-major, no swizzle
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (static_cast<uint64_t>((saddr & 0x3FFFFu) >> 4)) | (static_cast<uint64_t>(lbo >> 4) << 16) |
         (static_cast<uint64_t>(sbo >> 4) << 32) | (1ull << 46);
}

// kind::i8 instruction descriptor: D s32, A/B u8, both K-major, M = 128, N = 128
constexpr uint32_t kIdesc = (2u << 4) | (0u << 7) | (0u << 10) | (static_cast<uint32_t>(kN >> 3) << 17) |
                            (static_cast<uint32_t>(kM >> 4) << 24);

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(kIdesc), "r"(accumulate));
}

__device__ __forceinline__ void commit(uint32_t mbar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(mbar) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t mbar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}\n" ::"r"(mbar),
      "r"(parity)
      : "memory");
}

// The dot product is invariant under any permutation of K applied to both
// operands, so a 32-bit word is spread "strided": byte 4j + b of the word's
// 32-byte K slice holds bit 8b + j, i.e. spread byte word j = (x >> j) &
// 0x01010101 — 15 ALU ops per word instead of ~32 for bit k -> byte k. Rows and
// classes are staged by the same function, so every (row, class) pair is
// summed over the same bits.
__device__ __forceinline__ uint32_t spread_lane(uint32_t x, uint32_t j) { return (x >> j) & 0x01010101u; }

// one 32-bit word of row r -> K bytes 32*kw .. 32*kw+31 of the chunk, in the
// core-matrix layout: K byte k of row r at (r/8)*kSbo + (k/16)*128 + (r%8)*16 + k%16
constexpr uint32_t kSbo = (kKBytes / 16) * 128;  // bytes between 8-row groups
__device__ __forceinline__ void sts128(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}
// tile = shared-window address of the operand tile (the extern array is
// re-aligned through a generic pointer, so plain C++ stores would compile to
// generic ST instead of STS)
__device__ __forceinline__ void stage_word(uint32_t tile, uint32_t r, uint32_t kw, uint32_t x) {
  const uint32_t base = tile + (r >> 3) * kSbo + (r & 7u) * 16 + 2 * kw * 128;
  sts128(base, spread_lane(x, 0), spread_lane(x, 1), spread_lane(x, 2), spread_lane(x, 3));
  sts128(base + 128, spread_lane(x, 4), spread_lane(x, 5), spread_lane(x, 6), spread_lane(x, 7));
}

__device__ __forceinline__ void mbar_init(uint32_t mbar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(mbar), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint32_t mbar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(mbar) : "memory");
}
// 16- / 4-byte async global -> shared copy; src_bytes = 0 zero-fills
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async4(uint32_t dst, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
// arrive on mbar once every cp.async this thread issued so far has landed
__device__ __forceinline__ void cp_async_arrive(uint32_t mbar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(mbar) : "memory");
}
__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}

}  // namespace tc
}  // namespace hvb
