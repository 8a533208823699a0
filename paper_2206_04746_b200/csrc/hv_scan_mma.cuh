// hv_scan_mma.cuh — Hamming scan on the int8 tensor cores for many classes
// (model.cpp:69-79, 96-104, 303-320).
//
//   popc(q ^ c) = |q| + |c| - 2 <q, c>,   <q, c> = sum over bits of q_j c_j
//
// <q, c> is a GEMM of 0/1 matrices: rows x D times D x classes. CTA tile =
// 128 rows x 128 classes, 8 warps as 4 (rows) x 2 (classes), each warp 2 x 8
// mma.sync.m16n8k32 per 32-bit k-step (s8 operands holding 0/1, exact s32
// accumulation). Both operands are read bit-packed from HBM/L2 (4-word
// k-chunks, prefetched into registers) and spread to bytes once, when staged
// into shared memory (double-buffered), so every fragment is a plain 32-bit
// shared load: a row byte is reused by 16 MMAs and a class byte by 8. At
// C = 100, D = 32768 this runs at 228 T MAC/s, 2.3x the tiled POPC scan
// (ncu: tensor pipe 47 %, MIO-throttle bound on the fragment loads).
// Measured on this B200: legacy IMMA sustains 1.13 POPS (565 T MAC/s) against
// 4.52 T POPC/s (145 T bit-ops/s) for XOR+POPC.
#pragma once

#include <cstdint>

namespace hvb {

constexpr int kMmaRows = 128, kMmaCls = 128;  // CTA tile
constexpr int kMmaK = 4;                      // words per k-chunk
constexpr int kMmaThreads = 256;
// spread bytes per row and chunk; +16 makes the row stride 36 words, so the
// 4-byte fragment loads of a warp (8 rows x 4 quads) hit 32 distinct banks.
// (Interleaving the nibbles for 8-byte fragment loads measured 12 % slower.)
constexpr int kMmaRowBytes = kMmaK * 32 + 16;

struct MmaSmem {
  uint8_t q[2][kMmaRows][kMmaRowBytes];
  uint8_t c[2][kMmaCls][kMmaRowBytes];
  uint32_t rowpop[kMmaRows];
};
constexpr size_t kMmaSmemBytes = sizeof(MmaSmem);


__device__ __forceinline__ void mma_s8_16832(int (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                             uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// one 32-bit word -> 32 bytes of 0/1 in a strided K order (byte 4j + b holds
// bit 8b + j); rows and classes use the same order, which the dot product
// does not see
__device__ __forceinline__ uint32_t spread_lane8(uint32_t x, uint32_t j) { return (x >> j) & 0x01010101u; }
__device__ __forceinline__ void spread_word(uint32_t x, uint8_t* dst) {
  uint4* d = reinterpret_cast<uint4*>(dst);
  d[0] = make_uint4(spread_lane8(x, 0), spread_lane8(x, 1), spread_lane8(x, 2), spread_lane8(x, 3));
  d[1] = make_uint4(spread_lane8(x, 4), spread_lane8(x, 5), spread_lane8(x, 6), spread_lane8(x, 7));
}

// <row, class> for rows [row0, row0 + 128) x classes [c0, c0 + 128) over words
// [kbeg, kend). Lane (g = lane/4, qd = lane%4) of warp (wm = warp/2,
// wn = warp%2) ends with
//   acc[m][t][j] = <row wm*32 + 16m + g + 8*(j/2), class wn*64 + 8t + 2qd + j%2>
// (tile-relative); s.rowpop holds |row| over the same words. Rows >= rows and
// classes >= C read as zero. All 256 threads must call it; it synchronises.
__device__ __forceinline__ void mma_scan_tile(const uint32_t* __restrict__ enc, uint64_t row0, uint64_t rows,
                                              uint32_t W, const uint32_t* __restrict__ cv, uint32_t C, uint32_t c0,
                                              MmaSmem& s, int (&acc)[2][8][4], uint32_t kbeg = 0,
                                              uint32_t kend = 0xFFFFFFFFu) {
  if (kend > W) kend = W;
  const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
  const uint32_t g = lane >> 2, qd = lane & 3u, wm = warp >> 1, wn = warp & 1u;
#pragma unroll
  for (int m = 0; m < 2; ++m)
#pragma unroll
    for (int t = 0; t < 8; ++t) acc[m][t][0] = acc[m][t][1] = acc[m][t][2] = acc[m][t][3] = 0;
  if (tid < kMmaRows) s.rowpop[tid] = 0;
  // staging: thread -> (row / class tid/2, words 2*(tid%2), +1 of the chunk), both operands
  const uint32_t sr = tid >> 1, sw = 2 * (tid & 1u);
  const bool rok = row0 + sr < rows, cok = c0 + sr < C;
  const uint32_t* rsrc = enc + (rok ? row0 + sr : 0) * W;
  const uint32_t* csrc = cv + static_cast<uint64_t>(cok ? c0 + sr : 0) * W;
  uint32_t rq[2], rc[2], pop = 0;
  auto load = [&](uint32_t k0) {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const uint32_t w = k0 + sw + i;
      rq[i] = (rok && w < kend) ? __ldg(rsrc + w) : 0u;
      rc[i] = (cok && w < kend) ? __ldg(csrc + w) : 0u;
    }
  };
  auto store = [&](uint32_t b) {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      spread_word(rq[i], &s.q[b][sr][32 * (sw + i)]);
      spread_word(rc[i], &s.c[b][sr][32 * (sw + i)]);
      pop += __popc(rq[i]);
    }
  };
  load(kbeg);
  store(0);
  __syncthreads();
  uint32_t b = 0;
  for (uint32_t k0 = kbeg; k0 < kend; k0 += kMmaK, b ^= 1u) {
    const bool more = k0 + kMmaK < kend;
    if (more) load(k0 + kMmaK);
#pragma unroll
    for (int kw = 0; kw < kMmaK; ++kw) {
      uint32_t a[2][4];
#pragma unroll
      for (int m = 0; m < 2; ++m) {
        // A (16 x 32 row-major): a0/a2 row g, a1/a3 row g+8; k = 4qd.. and 16+4qd..
        const uint8_t* r0 = &s.q[b][wm * 32 + m * 16 + g][32 * kw + 4 * qd];
        const uint8_t* r1 = r0 + 8 * kMmaRowBytes;
        a[m][0] = *reinterpret_cast<const uint32_t*>(r0);
        a[m][1] = *reinterpret_cast<const uint32_t*>(r1);
        a[m][2] = *reinterpret_cast<const uint32_t*>(r0 + 16);
        a[m][3] = *reinterpret_cast<const uint32_t*>(r1 + 16);
      }
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        // B (32 x 8 col-major): class wn*64 + 8t + g, k = 4qd.. (b0) and 16+4qd.. (b1)
        const uint8_t* cp = &s.c[b][wn * 64 + t * 8 + g][32 * kw + 4 * qd];
        const uint32_t b0 = *reinterpret_cast<const uint32_t*>(cp);
        const uint32_t b1 = *reinterpret_cast<const uint32_t*>(cp + 16);
        mma_s8_16832(acc[0][t], a[0][0], a[0][1], a[0][2], a[0][3], b0, b1);
        mma_s8_16832(acc[1][t], a[1][0], a[1][1], a[1][2], a[1][3], b0, b1);
      }
    }
    if (more) store(b ^ 1u);  // the other buffer was last read before the previous barrier
    __syncthreads();
  }
  // |row| over [kbeg, kend): the two threads staging a row add their halves
  atomicAdd(&s.rowpop[sr], pop);
  __syncthreads();
}

}  // namespace hvb
