// hv_scan.cuh — CTA-tiled Hamming scan for many classes (model.cpp:69-79,
// 96-104, 303-320): popcount(row ^ class_vector) for a tile of 32 rows x 32
// classes, the words streamed through shared memory in double-buffered
// k-tiles of 64.
//
// Lane = class (so no cross-lane reduction per popcount), 8 compute warps x 4
// rows; per word a lane reads its class word (conflict-free, padded layout)
// and the 4 row words (broadcast), then issues 4 XOR+POPC+ADD. Loads of the
// next k-tile are in flight while the current one is counted. The scan is
// bound by the XU pipe (POPC, 16 lanes/clk/SM); a warp per query (the C < 32
// path) is latency-bound on re-reading every class vector per row instead.
#pragma once

#include <cstdint>

namespace hvb {

constexpr int kScanRows = 32;        // rows per tile (8 warps x 4)
constexpr int kScanCls = 32;         // classes per tile (lane = class)
constexpr int kScanK = 64;           // words per k-tile
constexpr int kScanRowsPerWarp = 4;

struct __align__(16) ScanSmem {
  uint32_t q[2][kScanRows][kScanK];        // row words
  uint32_t c[2][kScanK][kScanCls + 1];     // class words, transposed, padded
};

// Popcounts over words [kbeg, kend) of rows [row0, row0 + nrows) (row stride
// W, nrows <= 32) against classes [c0, c0 + 32) of cv (C x W). On return, lane l of warp w (w < 8)
// holds in a[k] the popcount of row row0 + 4w + k against class c0 + l (junk
// for rows/classes out of range). Every thread of the CTA must call it
// (blockDim.x >= 256); it synchronises the CTA.
template <int NT>
__device__ __forceinline__ void scan_tile(const uint32_t* __restrict__ rows, uint64_t row0, uint32_t nrows,
                                          uint32_t W, const uint32_t* __restrict__ cv, uint32_t C, uint32_t c0,
                                          ScanSmem& s, uint32_t (&a)[kScanRowsPerWarp], uint32_t kbeg = 0,
                                          uint32_t kend = 0xFFFFFFFFu) {
  if (kend > W) kend = W;
  constexpr int kQ = (kScanRows * kScanK + NT - 1) / NT;
  constexpr int kC = (kScanCls * kScanK + NT - 1) / NT;
  const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
#pragma unroll
  for (int k = 0; k < kScanRowsPerWarp; ++k) a[k] = 0;
  uint32_t rq[kQ], rc[kC];
  auto load = [&](uint32_t k0) {
#pragma unroll
    for (int i = 0; i < kQ; ++i) {
      const uint32_t e = tid + i * NT;
      const uint32_t r = e / kScanK, w = e % kScanK;
      rq[i] = (e < kScanRows * kScanK && r < nrows && k0 + w < kend) ? __ldg(rows + (row0 + r) * W + k0 + w) : 0u;
    }
#pragma unroll
    for (int i = 0; i < kC; ++i) {
      const uint32_t e = tid + i * NT;
      const uint32_t c = e / kScanK, w = e % kScanK;
      rc[i] = (e < kScanCls * kScanK && c0 + c < C && k0 + w < kend) ? cv[static_cast<uint64_t>(c0 + c) * W + k0 + w]
                                                                     : 0u;
    }
  };
  auto store = [&](uint32_t b) {
#pragma unroll
    for (int i = 0; i < kQ; ++i) {
      const uint32_t e = tid + i * NT;
      if (e < kScanRows * kScanK) s.q[b][e / kScanK][e % kScanK] = rq[i];
    }
#pragma unroll
    for (int i = 0; i < kC; ++i) {
      const uint32_t e = tid + i * NT;
      if (e < kScanCls * kScanK) s.c[b][e % kScanK][e / kScanK] = rc[i];
    }
  };
  load(kbeg);
  store(0);
  __syncthreads();
  uint32_t b = 0;
  for (uint32_t k0 = kbeg; k0 < kend; k0 += kScanK, b ^= 1u) {
    const bool more = k0 + kScanK < kend;
    if (more) load(k0 + kScanK);
    if (warp < kScanRows / kScanRowsPerWarp) {
      const uint32_t r0 = warp * kScanRowsPerWarp;
#pragma unroll 4
      for (int w = 0; w < kScanK; w += 4) {
        const uint32_t c0w = s.c[b][w][lane], c1w = s.c[b][w + 1][lane];
        const uint32_t c2w = s.c[b][w + 2][lane], c3w = s.c[b][w + 3][lane];
#pragma unroll
        for (int k = 0; k < kScanRowsPerWarp; ++k) {
          const uint4 q = *reinterpret_cast<const uint4*>(&s.q[b][r0 + k][w]);
          a[k] += __popc(q.x ^ c0w) + __popc(q.y ^ c1w) + __popc(q.z ^ c2w) + __popc(q.w ^ c3w);
        }
      }
    }
    if (more) store(b ^ 1u);  // last read before the previous barrier
    __syncthreads();
  }
}

// argmin key: popcount in the high word, class in the low word, so the
// minimum is the reference's strict-< argmin (lowest class on ties).
__device__ __forceinline__ unsigned long long scan_key(uint32_t popc, uint32_t c) {
  return (static_cast<unsigned long long>(popc) << 32) | c;
}

__device__ __forceinline__ unsigned long long warp_min_u64(unsigned long long key) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long other = __shfl_xor_sync(0xFFFFFFFFu, key, o);
    key = other < key ? other : key;
  }
  return key;
}

}  // namespace hvb
