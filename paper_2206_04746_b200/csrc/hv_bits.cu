// hv_bits.cu — packed bit-matrix kernels (reference kernels.hpp:16-63):
// pack / unpack / xor_bind / rotate / horizontal_sum / transpose /
// vertical_sum / majority_binarize, plus the shared column-count kernel that
// classical training also uses.
//
// All kernels are HBM-streaming integer work: coalesced 32-bit word access
// (a warp covers 128 contiguous bytes), grid-stride loops sized to the SM
// count, no shared-memory staging needed except where noted.

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "hv_internal.cuh"
#include "hv_scan_tc.cuh"

namespace hvb {

// --------------------------------------------------------------- pack ----
// kernels.cpp:44-73. HBM-streaming byte <-> bit conversions in two shapes:
//
// * rows of a multiple of 16 bytes (D = 1024, 10000, 20000, 32768 ...): a
//   thread owns 16 dense bytes = half a packed word. pack: one 128-bit load,
//   each 4-byte group of 0/1 bytes becomes 4 bits with one multiply (the
//   top byte of (x & 0x01010101) * 0x01020408 is b0 + 2 b1 + 4 b2 + 8 b3; the
//   lower partial products stay below 2^24), the 16 bits are stored as one
//   16-bit half of the output word. unpack: the inverse, a nibble spread to
//   4 bytes by (n * 0x00204081) & 0x01010101, one 128-bit store.
// * rows of a multiple of 4 bytes: 8 lanes per word, one 4-byte group each
//   (the same multiply), OR-reduced with 3 shuffles;
// * any other D: a warp per output word, lane l owns dense byte 32 w + l of
//   the row; pack = __ballot_sync of the bytes (32 coalesced byte loads), and
//   unpack = one bit per lane.
//
// Non-binary bytes latch the first (row-major) offending flat index, the
// reference's error (kernels.cpp:45-51).
__device__ __forceinline__ uint32_t nibble_of(uint32_t x) { return ((x & 0x01010101u) * 0x01020408u) >> 24; }
__device__ __forceinline__ uint32_t spread_nibble(uint32_t n) { return (n * 0x00204081u) & 0x01010101u; }

__global__ void pack16_kernel(const uint4* __restrict__ dense, uint64_t rows, uint32_t dim, uint32_t W,
                              uint16_t* __restrict__ out, unsigned long long* err) {
  const uint32_t per_row = dim / 16;  // 16-byte chunks per row
  const uint64_t total = rows * per_row;
  const bool odd_half = (dim % 32) != 0;  // the last word of a row has a zero high half
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint4 v = __ldcs(dense + i);
    const uint32_t bad = (v.x | v.y | v.z | v.w) & 0xFEFEFEFEu;
    if (bad) {  // rare: find the first non-binary byte of the chunk
      const uint32_t q[4] = {v.x, v.y, v.z, v.w};
      for (int k = 0; k < 4; ++k) {
        const uint32_t bk = q[k] & 0xFEFEFEFEu;
        if (bk) {
          latch(err, kErrByte, i * 16 + 4 * k + (__ffs(bk) - 1) / 8);
          break;
        }
      }
    }
    const uint32_t bits = nibble_of(v.x) | (nibble_of(v.y) << 4) | (nibble_of(v.z) << 8) | (nibble_of(v.w) << 12);
    const uint64_t r = i / per_row;
    const uint32_t c = static_cast<uint32_t>(i % per_row);  // half-word index within the row
    uint16_t* o = out + (r * W) * 2 + c;
    o[0] = static_cast<uint16_t>(bits);
    if (odd_half && c == per_row - 1) o[1] = 0;  // padding bits of the row's last word stay zero
  }
}

__global__ void unpack16_kernel(const uint16_t* __restrict__ words, uint64_t rows, uint32_t dim, uint32_t W,
                                uint4* __restrict__ dense) {
  const uint32_t per_row = dim / 16;
  const uint64_t total = rows * per_row;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t r = i / per_row;
    const uint32_t c = static_cast<uint32_t>(i % per_row);
    const uint32_t h = __ldg(words + (r * W) * 2 + c);
    __stcs(dense + i, make_uint4(spread_nibble(h & 15u), spread_nibble((h >> 4) & 15u), spread_nibble((h >> 8) & 15u),
                                 spread_nibble(h >> 12)));
  }
}

// Rows of a multiple of 4 bytes (D = 1000, 100 ...): 8 lanes per output
// word, each with one 4-byte group (4 bits), OR-reduced across the 8 lanes.
__global__ void pack4_kernel(const uint32_t* __restrict__ dense, uint64_t rows, uint32_t dim, uint32_t W,
                             uint32_t* __restrict__ out, unsigned long long* err) {
  const uint32_t k = threadIdx.x & 7u;  // 4-byte group within the word
  const uint32_t groups = dim / 4;
  const uint64_t total = rows * W;
  const uint64_t ngroups = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 3;
  for (uint64_t g = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 3; g < total; g += ngroups) {
    const uint64_t r = g / W;
    const uint32_t w = static_cast<uint32_t>(g % W);
    const uint32_t q = 8u * w + k;
    const uint32_t x = q < groups ? __ldcs(dense + r * groups + q) : 0u;
    const uint32_t badb = x & 0xFEFEFEFEu;
    if (badb) latch(err, kErrByte, r * dim + 4ull * q + (__ffs(badb) - 1) / 8);
    uint32_t v = nibble_of(x) << (4u * k);
    v |= __shfl_xor_sync(0xFFFFFFFFu, v, 1);
    v |= __shfl_xor_sync(0xFFFFFFFFu, v, 2);
    v |= __shfl_xor_sync(0xFFFFFFFFu, v, 4);
    if (k == 0) out[g] = v;
  }
}

__global__ void unpack4_kernel(const uint32_t* __restrict__ words, uint64_t rows, uint32_t dim, uint32_t W,
                               uint32_t* __restrict__ dense) {
  const uint32_t k = threadIdx.x & 7u;
  const uint32_t groups = dim / 4;
  const uint64_t total = rows * W;
  const uint64_t ngroups = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 3;
  for (uint64_t g = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 3; g < total; g += ngroups) {
    const uint64_t r = g / W;
    const uint32_t w = static_cast<uint32_t>(g % W);
    const uint32_t q = 8u * w + k;
    const uint32_t v = __ldg(words + g);
    if (q < groups) __stcs(dense + r * groups + q, spread_nibble((v >> (4u * k)) & 15u));
  }
}

__global__ void pack_ballot_kernel(const uint8_t* __restrict__ dense, uint64_t rows, uint32_t dim, uint32_t W,
                                   uint32_t* __restrict__ out, unsigned long long* err) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint64_t total = rows * W;
  const uint64_t nwarps = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t i = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; i < total; i += nwarps) {
    const uint64_t r = i / W;
    const uint32_t w = static_cast<uint32_t>(i % W);
    const uint32_t col = w * 32u + lane;
    const uint32_t b = col < dim ? dense[r * dim + col] : 0u;
    const uint32_t bad = __ballot_sync(0xFFFFFFFFu, b > 1u);
    if (bad && lane == 0) latch(err, kErrByte, r * dim + w * 32u + (__ffs(bad) - 1));
    const uint32_t word = __ballot_sync(0xFFFFFFFFu, b & 1u);
    if (lane == 0) out[i] = word;
  }
}

__global__ void unpack_ballot_kernel(const uint32_t* __restrict__ words, uint64_t rows, uint32_t dim, uint32_t W,
                                     uint8_t* __restrict__ dense) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint64_t total = rows * W;
  const uint64_t nwarps = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t i = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; i < total; i += nwarps) {
    const uint64_t r = i / W;
    const uint32_t w = static_cast<uint32_t>(i % W);
    const uint32_t v = __ldg(words + i);
    const uint32_t col = w * 32u + lane;
    if (col < dim) dense[r * dim + col] = static_cast<uint8_t>((v >> lane) & 1u);
  }
}

// kernels.cpp:75-87 (b broadcast when b_rows == 1)
__global__ void xor_kernel(const uint32_t* __restrict__ a, const uint32_t* __restrict__ b, uint64_t rows,
                           uint32_t W, bool broadcast, uint32_t* __restrict__ out) {
  const uint64_t total = rows * W;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
    out[i] = a[i] ^ b[broadcast ? (i % W) : i];
  }
}

// kernels.cpp:89-101: output bit (j + s) mod D = input bit j. Output word w
// gathers 32 bits starting at input position (32w - s) mod D, cyclically.
__global__ void rotate_kernel(const uint32_t* __restrict__ m, uint64_t rows, uint32_t dim, uint32_t W,
                              uint32_t s, uint32_t* __restrict__ out) {
  const uint64_t total = rows * W;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t r = i / W;
    const uint32_t w = static_cast<uint32_t>(i % W);
    const uint32_t p = static_cast<uint32_t>((static_cast<uint64_t>(w) * 32u + dim - s) % dim);
    out[i] = get_bits_cyclic(m + r * W, W, dim, p) & valid_mask(w, dim);
  }
}

// kernels.cpp:103-109. One warp per row.
__global__ void hsum_kernel(const uint32_t* __restrict__ m, uint64_t rows, uint32_t W, uint64_t* __restrict__ out) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x >> 5);
  for (uint64_t r = blockIdx.x * (uint64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); r < rows; r += warps) {
    uint32_t c = 0;
    for (uint32_t w = lane; w < W; w += 32u) c += __popc(m[r * W + w]);
    c = __reduce_add_sync(0xFFFFFFFFu, c);
    if (lane == 0) out[r] = c;
  }
}

// kernels.cpp:111-135. One warp per 32x32 tile: lane r holds row r's word,
// 32 ballots produce the 32 transposed words (lane t keeps ballot t).
__global__ void transpose_kernel(const uint32_t* __restrict__ m, uint32_t rows, uint32_t dim, uint32_t W,
                                 uint32_t outW, uint32_t* __restrict__ out) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint64_t tiles = static_cast<uint64_t>(outW) * W;
  const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x >> 5);
  for (uint64_t t = blockIdx.x * (uint64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); t < tiles; t += warps) {
    const uint32_t br = static_cast<uint32_t>(t / W);  // row block
    const uint32_t bc = static_cast<uint32_t>(t % W);  // column word
    const uint32_t row = br * 32u + lane;
    const uint32_t v = row < rows ? m[static_cast<uint64_t>(row) * W + bc] : 0u;
    uint32_t mine = 0;
#pragma unroll
    for (uint32_t k = 0; k < 32; ++k) {
      const uint32_t b = __ballot_sync(0xFFFFFFFFu, (v >> k) & 1u);
      if (lane == k) mine = b;
    }
    const uint32_t col = bc * 32u + lane;
    if (col < dim) out[static_cast<uint64_t>(col) * outW + br] = mine;
  }
}

// kernels.cpp:142-160
__global__ void majority_kernel(const uint64_t* __restrict__ counts, uint32_t dim, uint32_t W, uint64_t n,
                                const uint32_t* __restrict__ tiebreak, uint32_t* __restrict__ out,
                                unsigned long long* err) {
  for (uint32_t w = blockIdx.x * blockDim.x + threadIdx.x; w < W; w += gridDim.x * blockDim.x) {
    uint32_t word = 0;
    const uint32_t tie = tiebreak[w];
    const uint32_t nb = min(32u, dim - w * 32u);
    for (uint32_t t = 0; t < nb; ++t) {
      const uint64_t c = counts[w * 32u + t];
      if (c > n) latch(err, kErrCount, w * 32u + t);
      const uint64_t twice = 2 * c;
      const uint32_t bit = twice > n ? 1u : (twice < n ? 0u : ((tie >> t) & 1u));
      word |= bit << t;
    }
    out[w] = word;
  }
}

// Column counts over a (permuted, segmented) row sequence: for segment s,
// counts[s][j] += #rows p in segment s with bit j set. The row sequence is
// perm[p] (or p) for p in [0, seg_off[nseg]).
//
// Rows of pitch ldm words, any alignment (the reference's unpitched layout).
// Work item = (row chunk of `chunk` <= 2048 positions, so 12-bit counters
// suffice; group of 32 word columns), one warp per item; a lane owns one
// column. Rows are loaded 32 per batch: 32 independent 4-byte loads in flight
// per lane (unpitched rows are only 4-byte aligned at odd W, so wider loads
// are not available). The batch's 32 row indices are fetched by the warp (the
// next batch's while this one's rows are in flight) and broadcast with
// shuffles, so a row costs one shuffle + one address per lane. Each column
// accumulates in a bit-sliced Harley–Seal counter (2 LOP3 per word) and is
// flushed with atomics at segment and chunk ends. scripts/probe_stream.cu
// (CHB-MIT, 5.65 M class-sorted rows of random words): 32 rows x 1 column per
// lane 3.6-3.7 TB/s; 16 x 4 1.9; the round-1 thread-per-column grid 3.47.
// Pitched, 16-byte aligned rows take column_count_staged_kernel instead.
template <class CT>
__global__ void __launch_bounds__(128) column_count_kernel(const uint32_t* __restrict__ m, uint32_t W, uint32_t ldm,
                                                           const uint32_t* __restrict__ perm,
                                                           const uint64_t* __restrict__ seg_off, uint32_t nseg,
                                                           uint64_t npos_fallback, uint32_t chunk, CT* single,
                                                           CT* const* __restrict__ dsts, uint32_t ndst) {
  constexpr int R = 32;
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t groups = (W + 31) / 32;
  const uint64_t npos = seg_off ? seg_off[nseg] : npos_fallback;
  const uint64_t items = (npos + chunk - 1) / chunk * groups;
  const uint64_t nwarps = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
  const uint64_t stride = 32ull * W;
  for (uint64_t it = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; it < items; it += nwarps) {
    const uint32_t col = static_cast<uint32_t>(it % groups) * 32 + lane;
    const bool ok = col < W;
    uint64_t p0 = (it / groups) * chunk;
    const uint64_t p1 = min(npos, p0 + chunk);
    uint32_t s = 0;
    if (seg_off) {
      while (s + 1 < nseg && seg_off[s + 1] <= p0) ++s;
    }
    while (p0 < p1) {
      const uint64_t e = seg_off ? min(p1, seg_off[s + 1]) : p1;
      if (e > p0) {
        HSCounter<8> h;
        uint32_t n0 = 0;
        if (p0 + lane < e) n0 = perm ? __ldg(perm + p0 + lane) : static_cast<uint32_t>(p0 + lane);
        for (uint64_t p = p0; p < e; p += R) {
          const uint32_t c0 = n0;
          const uint32_t nvalid = e - p < R ? static_cast<uint32_t>(e - p) : static_cast<uint32_t>(R);
          const uint32_t* mc = m + col;
          uint32_t x[R];
#pragma unroll
          for (int t = 0; t < R; ++t) {
            const uint32_t r = __shfl_sync(0xFFFFFFFFu, c0, t);
            x[t] = (ok && t < nvalid) ? __ldcs(mc + static_cast<uint64_t>(r) * ldm) : 0u;
          }
          const uint64_t q = p + R + lane;
          if (q < e) n0 = perm ? __ldg(perm + q) : static_cast<uint32_t>(q);
#pragma unroll
          for (int j = 0; j < R; j += 16) h.add16(x + j);
        }
        // flush into every destination: the local counts, or — fused with the
        // all-reduce — the count buffers of all ranks over peer memory
        if (ok) {
          for (uint32_t d = 0; d < ndst; ++d) {
            CT* dst = (dsts ? dsts[d] : single) + s * stride + 32ull * col;
#pragma unroll 4
            for (int t = 0; t < 32; ++t) {
              const uint32_t c = h.count_of(t);
              if (c == 0) continue;
              if (ndst == 1) {
                atomicAdd(dst + t, static_cast<CT>(c));
              } else {
                atomicAdd_system(dst + t, static_cast<CT>(c));  // peer memory: system scope
              }
            }
          }
        }
      }
      p0 = e;
      ++s;
    }
  }
}

// Rows of pitch ldm % 4 == 0 words, 16-byte aligned (the engine's pitched
// layout): whole row segments are staged into shared memory by the bulk-copy
// (TMA) engine, so HBM sees each row as one contiguous read — the pattern
// that streams at ~6 TB/s here (scripts/probe_stream.cu), where per-warp
// 128-byte slices of 32 different rows stop at ~3.7.
// CTA = (column range [c0, c0 + ncols), ncols <= 512 words; row chunk of
// `chunk` positions). Thread j owns column c0 + j. kCsStages stages of
// kCsRows rows (default 2 x 16): warp 0 issues one cp.async.bulk per row (the row's columns
// c0 .. c0 + ncols rounded up to 16 bytes) completing on the stage's
// mbarrier (warp 0: a lane per row); every thread reads its column of each staged row (consecutive
// words: conflict-free), adds 16 rows at a time into its Harley–Seal
// counter, and arrives on the stage's `empty` barrier; warp 0 refills the
// stage when every warp has. Class segments inside a batch (at most C - 1 per
// call) split the batch.
constexpr int kCsMaxCols = 512;

template <class CT>
__device__ __forceinline__ void flush_counts(const HSCounter<8>& h, uint32_t col, uint64_t seg_stride, uint32_t s,
                                             CT* single, CT* const* __restrict__ dsts, uint32_t ndst) {
  for (uint32_t d = 0; d < ndst; ++d) {
    CT* dst = (dsts ? dsts[d] : single) + s * seg_stride + 32ull * col;
#pragma unroll 4
    for (int t = 0; t < 32; ++t) {
      const uint32_t c = h.count_of(t);
      if (c == 0) continue;
      if (ndst == 1) {
        atomicAdd(dst + t, static_cast<CT>(c));
      } else {
        atomicAdd_system(dst + t, static_cast<CT>(c));  // peer memory: system scope
      }
    }
  }
}

template <class CT, int kCsRows, int kCsStages>
__global__ void __launch_bounds__(kCsMaxCols) column_count_staged_kernel(
    const uint32_t* __restrict__ m, uint32_t W, uint32_t ldm, const uint32_t* __restrict__ perm,
    const uint64_t* __restrict__ seg_off, uint32_t nseg, uint64_t npos_fallback, uint32_t chunk, uint32_t ncols,
    CT* single, CT* const* __restrict__ dsts, uint32_t ndst) {
  extern __shared__ __align__(128) uint32_t cs_rows[];  // [stage][row][ncols]
  __shared__ __align__(8) unsigned long long full[kCsStages], empty[kCsStages];
  const uint32_t c0 = blockIdx.x * ncols;
  const uint32_t nc = min(ncols, W - c0);
  const uint32_t bytes = (nc + 3) / 4 * 16;
  const uint32_t j = threadIdx.x;
  const bool ok = j < nc;
  const uint32_t nwarps = blockDim.x >> 5;
  const uint64_t npos = seg_off ? seg_off[nseg] : npos_fallback;
  const uint64_t p0 = static_cast<uint64_t>(blockIdx.y) * chunk;
  if (p0 >= npos) return;
  const uint64_t p1 = min(npos, p0 + chunk);
  const uint32_t nbatch = static_cast<uint32_t>((p1 - p0 + kCsRows - 1) / kCsRows);
  const uint32_t sbase = tc::smem_u32(cs_rows);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int s = 0; s < kCsStages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(tc::smem_u32(&full[s])) : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(tc::smem_u32(&empty[s])), "r"(nwarps) : "memory");
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // warp 0 feeds the stages: lane t copies row t of a batch (one bulk copy per
  // lane, after lane 0 armed the stage's transaction count), and holds the
  // permutation entry of the next batch to issue, loaded one batch ahead. A
  // stage is refilled once every warp has arrived on its `empty` barrier.
  const uint32_t lane = threadIdx.x & 31u;
  uint32_t next_row = 0;
  auto load_rows = [&](uint32_t b) {
    const uint64_t q = p0 + static_cast<uint64_t>(b) * kCsRows + lane;
    if (b < nbatch && lane < kCsRows && q < p1) next_row = perm ? __ldg(perm + q) : static_cast<uint32_t>(q);
  };
  auto issue = [&](uint32_t b) {  // warp 0: stage b % kCsStages <- rows of batch b
    const uint32_t st = b % kCsStages;
    if (b >= static_cast<uint32_t>(kCsStages)) {
      tc::mbar_wait(tc::smem_u32(&empty[st]), (b / kCsStages - 1) & 1u);
    }
    const uint64_t pb = p0 + static_cast<uint64_t>(b) * kCsRows;
    const uint32_t n = p1 - pb < kCsRows ? static_cast<uint32_t>(p1 - pb) : static_cast<uint32_t>(kCsRows);
    const uint32_t mb = tc::smem_u32(&full[st]);
    if (lane == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(n * bytes) : "memory");
    }
    __syncwarp();
    if (lane < n) {
      const uint32_t dst = sbase + (st * kCsRows + lane) * ncols * 4u;
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                   "l"(m + static_cast<uint64_t>(next_row) * ldm + c0), "r"(bytes), "r"(mb)
                   : "memory");
    }
    load_rows(b + 1);
  };
  if (threadIdx.x < 32) {
    load_rows(0);
    for (uint32_t b = 0; b < nbatch && b < static_cast<uint32_t>(kCsStages); ++b) issue(b);
  }
  uint32_t s = 0;
  if (seg_off) {
    while (s + 1 < nseg && seg_off[s + 1] <= p0) ++s;
  }
  uint64_t seg_end = seg_off ? seg_off[s + 1] : npos;
  const uint64_t seg_stride = 32ull * W;
  const uint32_t jj = ok ? j : 0u;  // idle columns read column 0 (inside the stage), never flushed
  HSCounter<8> h;
  for (uint32_t b = 0; b < nbatch; ++b) {
    const uint32_t st = b % kCsStages;
    tc::mbar_wait(tc::smem_u32(&full[st]), (b / kCsStages) & 1u);
    const uint64_t pb = p0 + static_cast<uint64_t>(b) * kCsRows;
    const uint64_t be = min(p1, pb + kCsRows);
    const uint32_t* src = cs_rows + st * kCsRows * ncols + jj;
    if (be == pb + kCsRows && be <= seg_end) {
      // the common case: a full batch inside one class segment
      uint32_t x[kCsRows];
#pragma unroll
      for (int t = 0; t < kCsRows; ++t) x[t] = src[t * ncols];
      if constexpr (kCsRows == 8) {
        h.add8(x);
      } else {
        if constexpr (kCsRows == 8) {
          h.add8(x);
        } else {
#pragma unroll
          for (int t = 0; t < kCsRows; t += 16) h.add16(x + t);
        }
      }
      if (be == seg_end && be < p1) {
        if (ok) flush_counts(h, c0 + j, seg_stride, s, single, dsts, ndst);
        h = HSCounter<8>();
        do {
          ++s;
          seg_end = seg_off[s + 1];
        } while (seg_end <= be && s + 1 < nseg);
      }
    } else {
      uint64_t lo = pb;
      while (lo < be) {
        const uint64_t hi = min(be, seg_end);
        const uint32_t tlo = static_cast<uint32_t>(lo - pb), thi = static_cast<uint32_t>(hi - pb);
        uint32_t x[kCsRows];
#pragma unroll
        for (int t = 0; t < kCsRows; ++t) x[t] = (t >= tlo && t < thi) ? src[t * ncols] : 0u;
        if constexpr (kCsRows == 8) {
          h.add8(x);
        } else {
#pragma unroll
          for (int t = 0; t < kCsRows; t += 16) h.add16(x + t);
        }
        lo = hi;
        if (hi == seg_end && hi < p1) {  // class segment ends inside the chunk
          if (ok) flush_counts(h, c0 + j, seg_stride, s, single, dsts, ndst);
          h = HSCounter<8>();
          do {
            ++s;
            seg_end = seg_off[s + 1];
          } while (seg_end <= lo && s + 1 < nseg);
        }
      }
    }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_u32(&empty[st])) : "memory");
    if (threadIdx.x < 32 && b + kCsStages < nbatch) issue(b + kCsStages);
  }
  if (ok) flush_counts(h, c0 + j, seg_stride, s, single, dsts, ndst);
}

// Grid for column_count_kernel: one warp per item (the one-shot grid measured
// faster than a wave-balanced grid-stride one).
template <class CT>
unsigned column_count_grid(uint64_t npos, uint32_t W, uint32_t chunk) {
  const uint64_t items = (npos + chunk - 1) / chunk * ((W + 31) / 32);
  return static_cast<unsigned>(std::max<uint64_t>(1, (items + 3) / 4));
}

void launch_column_count_u32(cudaStream_t st, const uint32_t* m, uint32_t W, const uint32_t* perm,
                             const uint64_t* seg_off, uint32_t nseg, uint64_t max_pos, uint32_t* counts, uint32_t ldm) {
  launch_column_count_peers(st, m, W, perm, seg_off, nseg, max_pos, counts, nullptr, 1, ldm);
}

template <class CT>
void launch_column_count_any(cudaStream_t st, const uint32_t* m, uint32_t W, uint32_t ldm, const uint32_t* perm,
                             const uint64_t* seg_off, uint32_t nseg, uint64_t max_pos, CT* single,
                             CT* const* dsts_dev, uint32_t ndst) {
  if (max_pos == 0 || W == 0) return;
  if (max_pos > 0xFFFFFFFFull) invalid("class counts: more than 2^32 rows per call");
  if (ldm == 0) ldm = W;
  if (ldm < W) invalid("class counts: row pitch < words per row");
  uint32_t chunk = 2048;
  if (ldm % 4 == 0 && (reinterpret_cast<uintptr_t>(m) & 15u) == 0) {
    // pitched, 16-byte aligned rows: TMA-staged whole-row reads
    const uint32_t W4 = (W + 3) / 4 * 4;
    const uint32_t nranges = (W4 + kCsMaxCols - 1) / kCsMaxCols;
    // short inputs (an online bootstrap batch, small folds): shorter chunks so
    // there are ~2 CTAs per SM instead of a handful (1,024 rows at W = 1024
    // were 2 CTAs)
    static int sms = 0;
    if (sms == 0) {
      int dev = 0;
      ck(cudaGetDevice(&dev), "cudaGetDevice");
      ck(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "sm count");
    }
    const uint64_t want_ctas = 2ull * static_cast<uint64_t>(sms);
    if ((max_pos + chunk - 1) / chunk * nranges < want_ctas) {
      const uint64_t c = (max_pos * nranges + want_ctas - 1) / want_ctas;
      chunk = static_cast<uint32_t>(std::max<uint64_t>(64, (c + 15) / 16 * 16));
    }
    const uint32_t ncols = (W4 / 4 + nranges - 1) / nranges * 4;  // balanced ranges, multiple of 4
    const uint32_t threads = (ncols + 31) / 32 * 32;
    dim3 grid(nranges, static_cast<unsigned>((max_pos + chunk - 1) / chunk));
    // 16 rows x 2 stages (40 KB: 5 CTAs per SM) measured best at CHB-MIT, 5.65 M
    // rows: 1.42 ms = 5.0 TB/s; 16 x 3 1.47, 32 x 2 1.50, 16 x 4 1.71, 8 x 4
    // 1.78, 16 x 6 3.06 (1 CTA per SM) — CTAs per SM matter more than depth
    int rows_per_stage = 16, stages = 2;
    if (const char* e = getenv("HVB200_CS_SHAPE")) sscanf(e, "%d,%d", &rows_per_stage, &stages);  // tuning
    auto go = [&](auto kern, int R, int S) {
      const size_t smem = static_cast<size_t>(S) * R * ncols * 4;
      ck(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)),
         "cudaFuncSetAttribute");
      kern<<<grid, threads, smem, st>>>(m, W, ldm, perm, seg_off, nseg, max_pos, chunk, ncols, single, dsts_dev,
                                        dsts_dev ? ndst : 1u);
    };
#define HV_CS(R, S)                                   \
  if (rows_per_stage == R && stages == S) {           \
    go(column_count_staged_kernel<CT, R, S>, R, S);   \
    launched("column_count_staged_kernel");           \
    return;                                           \
  }
    HV_CS(8, 4) HV_CS(16, 3) HV_CS(16, 4) HV_CS(32, 2)
#undef HV_CS
    go(column_count_staged_kernel<CT, 16, 2>, 16, 2);
    launched("column_count_staged_kernel");
    return;
  }
  {  // short inputs: shorter chunks for ~8 warps per SM
    static int sms2 = 0;
    if (sms2 == 0) {
      int dev = 0;
      ck(cudaGetDevice(&dev), "cudaGetDevice");
      ck(cudaDeviceGetAttribute(&sms2, cudaDevAttrMultiProcessorCount, dev), "sm count");
    }
    const uint64_t groups = (W + 31) / 32, want_warps = 8ull * static_cast<uint64_t>(sms2);
    if ((max_pos + chunk - 1) / chunk * groups < want_warps) {
      const uint64_t c = (max_pos * groups + want_warps - 1) / want_warps;
      chunk = static_cast<uint32_t>(std::max<uint64_t>(64, (c + 31) / 32 * 32));
    }
  }
  const unsigned grid = column_count_grid<CT>(max_pos, W, chunk);
  column_count_kernel<CT><<<grid, 128, 0, st>>>(m, W, ldm, perm, seg_off, nseg, max_pos, chunk, single, dsts_dev,
                                                dsts_dev ? ndst : 1u);
  launched("column_count_kernel");
}

void launch_column_count_peers(cudaStream_t st, const uint32_t* m, uint32_t W, const uint32_t* perm,
                               const uint64_t* seg_off, uint32_t nseg, uint64_t max_pos, uint32_t* single,
                               uint32_t* const* dsts_dev, uint32_t ndst, uint32_t ldm) {
  launch_column_count_any<uint32_t>(st, m, W, ldm, perm, seg_off, nseg, max_pos, single, dsts_dev, ndst);
}

__global__ void widen_u64_kernel(const unsigned long long* __restrict__ in, uint32_t dim, uint64_t* __restrict__ out) {
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < dim; j += gridDim.x * blockDim.x) out[j] = in[j];
}

}  // namespace hvb

using namespace hvb;

namespace {

unsigned stream_grid(hv_context* ctx, uint64_t items, unsigned block) {
  const uint64_t want = (items + block - 1) / block;
  const uint64_t cap = static_cast<uint64_t>(ctx->sm_count) * 8;
  return static_cast<unsigned>(want == 0 ? 1 : (want < cap ? want : cap));
}

void pack_device(hv_context* ctx, cudaStream_t st, const uint8_t* dense, size_t rows, size_t dim, uint32_t* out) {
  const size_t W = words_per_row(dim);
  if (rows * W == 0) return;
  if (dim % 16 == 0 && (reinterpret_cast<uintptr_t>(dense) & 15u) == 0) {
    pack16_kernel<<<stream_grid(ctx, rows * (dim / 16), 256), 256, 0, st>>>(
        reinterpret_cast<const uint4*>(dense), rows, static_cast<uint32_t>(dim), static_cast<uint32_t>(W),
        reinterpret_cast<uint16_t*>(out), ctx->d_err);
    launched("pack16_kernel");
  } else if (dim % 4 == 0 && (reinterpret_cast<uintptr_t>(dense) & 3u) == 0) {
    pack4_kernel<<<stream_grid(ctx, rows * W * 8, 256), 256, 0, st>>>(
        reinterpret_cast<const uint32_t*>(dense), rows, static_cast<uint32_t>(dim), static_cast<uint32_t>(W), out,
        ctx->d_err);
    launched("pack4_kernel");
  } else {
    pack_ballot_kernel<<<stream_grid(ctx, rows * W * 32, 256), 256, 0, st>>>(dense, rows, static_cast<uint32_t>(dim),
                                                                           static_cast<uint32_t>(W), out, ctx->d_err);
    launched("pack_ballot_kernel");
  }
}

void unpack_device(hv_context* ctx, cudaStream_t st, const uint32_t* words, size_t rows, size_t dim, uint8_t* dense) {
  const size_t W = words_per_row(dim);
  if (rows * W == 0) return;
  if (dim % 16 == 0 && (reinterpret_cast<uintptr_t>(dense) & 15u) == 0) {
    unpack16_kernel<<<stream_grid(ctx, rows * (dim / 16), 256), 256, 0, st>>>(
        reinterpret_cast<const uint16_t*>(words), rows, static_cast<uint32_t>(dim), static_cast<uint32_t>(W),
        reinterpret_cast<uint4*>(dense));
    launched("unpack16_kernel");
  } else if (dim % 4 == 0 && (reinterpret_cast<uintptr_t>(dense) & 3u) == 0) {
    unpack4_kernel<<<stream_grid(ctx, rows * W * 8, 256), 256, 0, st>>>(
        words, rows, static_cast<uint32_t>(dim), static_cast<uint32_t>(W), reinterpret_cast<uint32_t*>(dense));
    launched("unpack4_kernel");
  } else {
    unpack_ballot_kernel<<<stream_grid(ctx, rows * W * 32, 256), 256, 0, st>>>(
        words, rows, static_cast<uint32_t>(dim), static_cast<uint32_t>(W), dense);
    launched("unpack_ballot_kernel");
  }
}

void check_latch(hv_context* ctx, const uint8_t* dense) {
  unsigned long long l[kErrKinds];
  read_latch(ctx, l);
  if (l[kErrByte] != ~0ull) {
    reset_latch(ctx);
    invalid("pack: non-binary entry " + std::to_string(int(dense[l[kErrByte]])) + " at flat index " +
            std::to_string(l[kErrByte]));
  }
}

}  // namespace

extern "C" {

hv_status hv_pack(hv_context* ctx, const uint8_t* dense, size_t rows, size_t dim, uint32_t* out) {
  return guarded([&] {
    require(ctx);
    const size_t W = words_per_row(dim);
    if (rows * W == 0) return;
    DevBuf<uint8_t> d_in(rows * dim, ctx->stream);
    DevBuf<uint32_t> d_out(rows * W, ctx->stream);
    d_in.upload(dense);
    pack_device(ctx, ctx->stream, d_in.ptr, rows, dim, d_out.ptr);
    d_out.download(out);
    check_latch(ctx, dense);
  });
}

hv_status hv_unpack(hv_context* ctx, const uint32_t* words, size_t rows, size_t dim, uint8_t* out) {
  return guarded([&] {
    require(ctx);
    const size_t W = words_per_row(dim);
    if (rows * W == 0) return;
    DevBuf<uint32_t> d_in(rows * W, ctx->stream);
    DevBuf<uint8_t> d_out(rows * dim, ctx->stream);
    d_in.upload(words);
    unpack_device(ctx, ctx->stream, d_in.ptr, rows, dim, d_out.ptr);
    d_out.download(out);
    sync(ctx);
  });
}

hv_status hv_xor_bind(hv_context* ctx, const uint32_t* a, size_t a_rows, size_t a_dim, const uint32_t* b,
                      size_t b_rows, size_t b_dim, uint32_t* out) {
  return guarded([&] {
    require(ctx);
    if (a_dim != b_dim || (b_rows != a_rows && b_rows != 1)) {
      invalid("xor_bind: shape mismatch (" + std::to_string(a_rows) + "x" + std::to_string(a_dim) + " vs " +
              std::to_string(b_rows) + "x" + std::to_string(b_dim) + ")");
    }
    const size_t W = words_per_row(a_dim);
    if (a_rows * W == 0) return;
    DevBuf<uint32_t> da(a_rows * W, ctx->stream), db(b_rows * W, ctx->stream), d_out(a_rows * W, ctx->stream);
    da.upload(a);
    db.upload(b);
    xor_kernel<<<stream_grid(ctx, a_rows * W, 256), 256, 0, ctx->stream>>>(da.ptr, db.ptr, a_rows, W,
                                                                          b_rows == 1 && a_rows != 1, d_out.ptr);
    launched("xor_kernel");
    d_out.download(out);
    sync(ctx);
  });
}

hv_status hv_rotate(hv_context* ctx, const uint32_t* m, size_t rows, size_t dim, size_t shift, uint32_t* out) {
  return guarded([&] {
    require(ctx);
    const size_t W = words_per_row(dim);
    if (rows * W == 0) return;
    const size_t s = dim == 0 ? 0 : shift % dim;
    if (s == 0) {
      std::copy(m, m + rows * W, out);
      return;
    }
    DevBuf<uint32_t> d_in(rows * W, ctx->stream), d_out(rows * W, ctx->stream);
    d_in.upload(m);
    rotate_kernel<<<stream_grid(ctx, rows * W, 256), 256, 0, ctx->stream>>>(d_in.ptr, rows, dim, W,
                                                                            static_cast<uint32_t>(s), d_out.ptr);
    launched("rotate_kernel");
    d_out.download(out);
    sync(ctx);
  });
}

hv_status hv_horizontal_sum(hv_context* ctx, const uint32_t* m, size_t rows, size_t dim, uint64_t* out) {
  return guarded([&] {
    require(ctx);
    const size_t W = words_per_row(dim);
    if (rows == 0) return;
    if (W == 0) {
      std::fill(out, out + rows, 0ull);
      return;
    }
    DevBuf<uint32_t> d_in(rows * W, ctx->stream);
    DevBuf<uint64_t> d_out(rows, ctx->stream);
    d_in.upload(m);
    hsum_kernel<<<stream_grid(ctx, rows * 32, 256), 256, 0, ctx->stream>>>(d_in.ptr, rows, W, d_out.ptr);
    launched("hsum_kernel");
    d_out.download(out);
    sync(ctx);
  });
}

hv_status hv_transpose(hv_context* ctx, const uint32_t* m, size_t rows, size_t dim, uint32_t* out) {
  return guarded([&] {
    require(ctx);
    const size_t W = words_per_row(dim);
    const size_t outW = words_per_row(rows);
    if (W == 0 || outW == 0) return;
    if (rows > 0xFFFFFFFFull || dim > 0xFFFFFFFFull) invalid("transpose: matrix too large");
    DevBuf<uint32_t> d_in(rows * W, ctx->stream), d_out(dim * outW, ctx->stream);
    d_in.upload(m);
    transpose_kernel<<<stream_grid(ctx, outW * W * 32, 256), 256, 0, ctx->stream>>>(
        d_in.ptr, static_cast<uint32_t>(rows), static_cast<uint32_t>(dim), W, outW, d_out.ptr);
    launched("transpose_kernel");
    d_out.download(out);
    sync(ctx);
  });
}

hv_status hv_vertical_sum(hv_context* ctx, const uint32_t* m, size_t rows, size_t dim, uint64_t* out) {
  return guarded([&] {
    require(ctx);
    const size_t W = words_per_row(dim);
    if (dim == 0) return;
    if (rows == 0) {
      std::fill(out, out + dim, 0ull);
      return;
    }
    DevBuf<uint32_t> d_in(rows * W, ctx->stream);
    DevBuf<unsigned long long> d_cnt(32 * W, ctx->stream);
    DevBuf<uint64_t> d_out(dim, ctx->stream);
    d_in.upload(m);
    d_cnt.zero();
    if (rows > 0xFFFFFFFFull) invalid("vertical_sum: more than 2^32 rows");
    launch_column_count_any<unsigned long long>(ctx->stream, d_in.ptr, W, W, nullptr, nullptr, 1, rows, d_cnt.ptr,
                                                nullptr, 1);
    widen_u64_kernel<<<grid_for(dim, 256), 256, 0, ctx->stream>>>(d_cnt.ptr, dim, d_out.ptr);
    launched("widen_u64_kernel");
    d_out.download(out);
    sync(ctx);
  });
}

hv_status hv_majority_binarize(hv_context* ctx, const uint64_t* counts, size_t dim, uint64_t n,
                               const uint32_t* tiebreak, size_t tiebreak_rows, size_t tiebreak_dim, uint32_t* out) {
  return guarded([&] {
    require(ctx);
    if (tiebreak_rows != 1 || tiebreak_dim != dim) {
      invalid("majority_binarize: tiebreak must be 1x" + std::to_string(dim));
    }
    const size_t W = words_per_row(dim);
    if (W == 0) return;
    DevBuf<uint64_t> d_c(dim, ctx->stream);
    DevBuf<uint32_t> d_t(W, ctx->stream), d_out(W, ctx->stream);
    d_c.upload(counts);
    d_t.upload(tiebreak);
    majority_kernel<<<grid_for(W, 128), 128, 0, ctx->stream>>>(d_c.ptr, dim, W, n, d_t.ptr, d_out.ptr, ctx->d_err);
    launched("majority_kernel");
    d_out.download(out);
    unsigned long long l[kErrKinds];
    read_latch(ctx, l);
    if (l[kErrCount] != ~0ull) {
      reset_latch(ctx);
      const size_t j = l[kErrCount];
      invalid("majority_binarize: count " + std::to_string(counts[j]) + " exceeds total " + std::to_string(n) +
              " at position " + std::to_string(j));
    }
  });
}

}  // extern "C"
