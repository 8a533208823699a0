// hv_scan_tc.cuh — the many-class Hamming scan on the 5th-generation tensor
// cores (tcgen05, kind::i8, accumulators in TMEM).
//
//   popc(q ^ c) = |q| + |c| - 2 <q, c>
//
// CTA tile = 128 rows x 128 classes; the K dimension is the hypervector's bits,
// 256 per chunk (8 words). 256 threads: thread t stages half of row t%128 and
// of class t%128 — the packed words of the next chunk are loaded into
// registers while the current chunk's MMAs run, then every bit is spread to a
// byte (0/1) and stored in the UMMA K-major no-swizzle layout (8-row x 16-byte core
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
constexpr uint32_t kTileBytes = kM * kKBytes;  // 16 KB per operand and stage

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

// 4 bits -> 4 bytes of 0/1: bit i of the nibble lands in byte i
__device__ __forceinline__ uint32_t spread4(uint32_t nib) { return (nib * 0x00204081u) & 0x01010101u; }

// one 32-bit word of row r -> bytes k = 32*kw .. 32*kw+31 of the chunk, in the
// core-matrix layout: byte k of row r at (r/8)*kSbo + (k/16)*128 + (r%8)*16 + k%16
constexpr uint32_t kSbo = (kKBytes / 16) * 128;  // bytes between 8-row groups
__device__ __forceinline__ void stage_word(uint8_t* tile, uint32_t r, uint32_t kw, uint32_t x) {
  uint8_t* base = tile + (r >> 3) * kSbo + (r & 7u) * 16;
  uint4* lo = reinterpret_cast<uint4*>(base + (2 * kw) * 128);
  uint4* hi = reinterpret_cast<uint4*>(base + (2 * kw + 1) * 128);
  *lo = make_uint4(spread4(x & 0xFu), spread4((x >> 4) & 0xFu), spread4((x >> 8) & 0xFu), spread4((x >> 12) & 0xFu));
  *hi = make_uint4(spread4((x >> 16) & 0xFu), spread4((x >> 20) & 0xFu), spread4((x >> 24) & 0xFu), spread4(x >> 28));
}

}  // namespace tc
}  // namespace hvb
