// hv_online.cu — the online trainer (model.cpp:250-301, Hamming metric) as
// ONE persistent cooperative kernel over all batches.
//
// The trainer is a chain of dependent batches: batch b is scored against the
// class vectors left by batch b-1, and every fp64 accumulator element must see
// the reference's sample-ordered in-place additions (model.cpp:54-63) to stay
// bit-identical. Per batch the work is small and latency-bound (CHB-MIT:
// 1,024 rows, two classes), so three kernel launches per batch with
// L2-latency-bound replays cost 180 us per batch (profiles/configs_r1.jsonl).
// Here one cooperative launch runs every batch, phases separated by grid.sync:
//
// score   (all warps)  per row: Hamming popcount against every class vector,
//         argmin (strict <, lowest class on ties, model.cpp:96-104) packed as
//         best = popc << 32 | class, plus the true class's popcount.
//         C < 16: warp per row, lanes over words. C >= 16: CTA-tiled scan
//         (hv_scan.cuh: 32 rows x 32 classes per tile, lane = class, words
//         through shared memory), per-row argmin merged across class blocks
//         with a 64-bit atomicMin.
//
// Two classes (C <= kMergedMaxC) or batches of <= 32 rows — MERGED:
//   replay  item = (class c, 32-word block, 4 bit columns per thread): the
//           batch is streamed in 64-row chunks; each chunk's labels/scores and the 8 words of every row
//           are loaded one chunk ahead into registers (the next chunk's loads
//           fly while this chunk is replayed), thread j replays the chunk's
//           entries of class c in row order on its register-held acc[c][j]
//           (delta_true for y == c, -gamma (1 - delta_pred) for pred == c != y),
//           a ninth warp advances the class weight over the true samples in
//           the same order. Class weights are double-buffered per batch parity
//           (every item of the class computes the same chain; word block 0
//           publishes it).
// Many classes — LISTS:
//   lists   CTA per class: the batch's entries compacted in row order (block
//           ballot + prefix) into a global list, weight chain, sample counts.
//   replay  item = (class, 32-word block) over its own list only (classes
//           untouched by the batch are skipped), chunks prefetched as above.
//
// Touched classes are re-binarised with the batch's final weight
// (model.cpp:139-163, 277-279).
#include <cooperative_groups.h>
#include <cuda_pipeline.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "hv_internal.cuh"
#include "hv_scan.cuh"

namespace cg = cooperative_groups;

namespace hvb {
namespace {

constexpr uint32_t kFull = 0xFFFFFFFFu;
#ifndef HV_REPLAY_UNROLL
#define HV_REPLAY_UNROLL 32  // COLS = 1 replay loop unroll: 4 / 8 / 16 / 32 -> 17.0 / 15.5 / 13.4 / 13.0 us per CHB-MIT batch
#endif
// A replay item is (class, block of 8*COLS words); each of its 256 replay
// threads owns COLS bit columns (independent accumulator chains) and the
// staged tile holds 256/COLS entries x 8*COLS words (2,048 words) either way.
// COLS = 1 suits long per-class lists (the chain length binds: fewer, longer
// chunks), COLS = 4 short ones (many classes: 4x fewer items per batch).
constexpr int kOReplay = 256;               // replay threads
constexpr int kOThreads = kOReplay + 32;    // + one warp for the weight chain
constexpr int kOTile = 2048;                // staged words per chunk
constexpr int kLChunk = 256;                // rows per compaction chunk (list building)
constexpr int kLoadsPer = (kOTile + kOThreads - 1) / kOThreads;  // word loads per thread per chunk
template <int COLS>
struct RTile {
  static constexpr int kWords = 8 * COLS;         // words per item
  static constexpr int kChunk = kOTile / kWords;  // entries per chunk
};
// COLS = 1 stages a chunk word-major: word ww of row k at ww * kWordPitch + k
// (pitch 260 = 256 rows + 4: 16-byte aligned for LDS.128, and the 8 words of
// one row land in 8 different banks when stored)
constexpr uint32_t kWordPitch = 260;
template <int COLS>
__device__ __forceinline__ uint32_t staged_word(uint32_t k, uint32_t ww) {
  return COLS == 1 ? ww * kWordPitch + k : k * RTile<COLS>::kWords + ww;
}
constexpr uint32_t kOrderMax = 1024;  // classes ordered longest-list-first when C <= this
constexpr uint32_t kMergedMaxC = 2;  // more classes: per-class lists skip the other classes' rows
constexpr uint32_t kLaneClassMinC = 16;  // measured: tiled wins at C = 26 (25 -> 17 us), loses at C <= 10

struct OnlineParams {
  const uint32_t* enc;
  const int32_t* labels;
  uint64_t rows;
  uint32_t D, W, C;
  uint64_t bsz;
  double gamma;
  const uint32_t* tie;
  double* acc;                 // C x D
  double* weight;              // 2 x C (MERGED: batch-parity ping-pong; LISTS: row 0)
  uint64_t* counts;            // C
  uint32_t* cv;                // C x W
  unsigned long long* best;    // 2 x bsz (batch parity): popc << 32 | class
  uint32_t* truep;             // bsz
  uint32_t* lidx;              // C x bsz (LISTS)
  double* lval;                // C x bsz (LISTS)
  uint32_t* llen;              // C (LISTS)
  unsigned long long* prof;    // optional: ns spent per phase (score, lists, replay), CTA 0's view
  uint32_t tiled;              // score with the CTA-tiled scan (lane = class) instead of warp per row
  uint32_t ksplit;             // tiled scoring: word range split into this many items per tile
  uint32_t* pscr;              // bsz x C partial popcounts (ksplit > 1), zero between batches
  uint32_t* arrive;            // per (row tile, class block) arrival counters (ksplit > 1)
  uint32_t* pre;               // optional: bsz x C popcounts of the (single) batch, precomputed;
                               // zeroed as read, and best[0, bsz) is reset after the batch
  uint32_t* wflag;             // MERGED: per-class epoch flags of the separate weight tasks (nullable)
  uint32_t* item_ctr;          // LISTS: dynamic replay-item counter (nullable: static round robin)
  uint32_t ablate;             // timing experiments only (HVB200_ONLINE_ABLATE): bit0 no next-chunk loads,
                               // bit1 no replay loop, bit2 no chunk stores (results are wrong)
  uint32_t mw;                 // MERGED: words per replay item (4: replay_merged_mw; 8: replay_merged)
};

__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* ptr) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ptr) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_u32(uint32_t* ptr, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(ptr), "r"(v) : "memory");
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ double delta_of(uint32_t popc, uint32_t D) {
  return static_cast<double>(popc) / static_cast<double>(D);  // model.cpp:69-79 (IEEE division)
}

__device__ __forceinline__ double penalty_of(unsigned long long best, double gamma, uint32_t D) {
  return __dmul_rn(-gamma, __dsub_rn(1.0, delta_of(static_cast<uint32_t>(best >> 32), D)));
}

// ---------------------------------------------------------------- score ----
// short rows (W <= 64) and up to kWarpC classes: the row word is loaded once
// per step and every class's word of that step is in flight together (one
// accumulator per class, reduced at the end) instead of one latency-bound
// pass per class. Measured: MNIST-shaped D = 1024 score phase 5.1 -> 2.9 us
// per batch; slower for long rows (D = 10000: 11.8 -> 14.6), which keep the
// per-class passes.
constexpr uint32_t kWarpC = 16;

template <uint32_t CM>
__device__ __forceinline__ void score_rows_all_classes(const OnlineParams& p, unsigned long long* best_out, uint64_t b0,
                                                       uint32_t n, uint64_t gwarp, uint64_t gwarps, uint32_t lane) {
  for (uint64_t r = gwarp; r < n; r += gwarps) {
    const uint32_t* q = p.enc + (b0 + r) * p.W;
    const int32_t y = p.labels[b0 + r];
    uint32_t a[CM];
#pragma unroll
    for (uint32_t c = 0; c < CM; ++c) a[c] = 0;
#pragma unroll 2
    for (uint32_t w = lane; w < p.W; w += 32u) {
      const uint32_t x = __ldg(q + w);
#pragma unroll
      for (uint32_t c = 0; c < CM; ++c) {
        if (c < p.C) a[c] += __popc(x ^ p.cv[static_cast<uint64_t>(c) * p.W + w]);
      }
    }
    uint32_t best = 0, bestp = kFull, truep = 0;
#pragma unroll
    for (uint32_t c = 0; c < CM; ++c) {
      if (c < p.C) {
        const uint32_t t = __reduce_add_sync(kFull, a[c]);
        if (t < bestp) {  // strict: the lowest class wins ties (model.cpp:96-104)
          bestp = t;
          best = c;
        }
        if (static_cast<int32_t>(c) == y) truep = t;
      }
    }
    if (lane == 0) {
      best_out[r] = (static_cast<unsigned long long>(bestp) << 32) | best;
      p.truep[r] = truep;
    }
  }
}

__device__ void score_warp_per_row(const OnlineParams& p, unsigned long long* best_out, uint64_t b0, uint32_t n,
                                   uint64_t gwarp, uint64_t gwarps, uint32_t lane) {
  // 3..16 classes, long rows whose words do not split evenly over the lanes:
  // every class's word of a step in flight together (per batch of 1,024:
  // UCI-HAR C = 6 18.4 -> 16.2 us, MNIST C = 10 D = 10000 29.8 -> 26.7 us);
  // rows of a multiple of 32 words keep the per-class passes (MNIST D = 8192
  // 23.4 vs 24.2, D = 16384 33.0 vs 34.9 us); two classes have their own
  // all-words-in-flight loop below (CHB-MIT: this path was 20.5 vs 18.2 us)
  const bool ragged = (p.W & 31u) != 0 && !(p.ablate & 64u);
  if (p.C >= 3 && p.C <= 8 && p.W > 64 && ragged) {
    score_rows_all_classes<8>(p, best_out, b0, n, gwarp, gwarps, lane);
    return;
  }
  if (p.C > 8 && p.C <= kWarpC && p.W > 64 && ragged) {
    score_rows_all_classes<kWarpC>(p, best_out, b0, n, gwarp, gwarps, lane);
    return;
  }
  if (p.C <= kWarpC && p.W <= 64) {
    for (uint64_t r = gwarp; r < n; r += gwarps) {
      const uint32_t* q = p.enc + (b0 + r) * p.W;
      const int32_t y = p.labels[b0 + r];
      uint32_t a[kWarpC];
#pragma unroll
      for (uint32_t c = 0; c < kWarpC; ++c) a[c] = 0;
      for (uint32_t w = lane; w < p.W; w += 32u) {
        const uint32_t x = __ldg(q + w);
#pragma unroll
        for (uint32_t c = 0; c < kWarpC; ++c) {
          if (c < p.C) a[c] += __popc(x ^ p.cv[static_cast<uint64_t>(c) * p.W + w]);
        }
      }
      uint32_t best = 0, bestp = kFull, truep = 0;
#pragma unroll
      for (uint32_t c = 0; c < kWarpC; ++c) {
        if (c < p.C) {
          const uint32_t t = __reduce_add_sync(kFull, a[c]);
          if (t < bestp) {  // strict: the lowest class wins ties (model.cpp:96-104)
            bestp = t;
            best = c;
          }
          if (static_cast<int32_t>(c) == y) truep = t;
        }
      }
      if (lane == 0) {
        best_out[r] = (static_cast<unsigned long long>(bestp) << 32) | best;
        p.truep[r] = truep;
      }
    }
    return;
  }
  if (p.C == 2 && p.W <= 32u * 10u && !(p.ablate & 4096u)) {
    // two classes (CHB-MIT W = 313): the row's and both class vectors' words
    // of every step loaded up front, one L2 round trip per row
    for (uint64_t r = gwarp; r < n; r += gwarps) {
      const uint32_t* q = p.enc + (b0 + r) * p.W;
      const int32_t y = p.labels[b0 + r];
      uint32_t x[10], v0[10], v1[10];
#pragma unroll
      for (int i = 0; i < 10; ++i) {
        const uint32_t w = lane + 32u * i;
        const bool ok = w < p.W;
        x[i] = ok ? __ldg(q + w) : 0u;
        v0[i] = ok ? p.cv[w] : 0u;
        v1[i] = ok ? p.cv[p.W + w] : 0u;
      }
      uint32_t a0 = 0, a1 = 0;
#pragma unroll
      for (int i = 0; i < 10; ++i) {
        a0 += __popc(x[i] ^ v0[i]);
        a1 += __popc(x[i] ^ v1[i]);
      }
      a0 = __reduce_add_sync(kFull, a0);
      a1 = __reduce_add_sync(kFull, a1);
      if (lane == 0) {
        const uint32_t best = a1 < a0 ? 1u : 0u;  // strict: class 0 wins ties (model.cpp:96-104)
        best_out[r] = (static_cast<unsigned long long>(best ? a1 : a0) << 32) | best;
        p.truep[r] = y == 1 ? a1 : (y == 0 ? a0 : 0u);
      }
    }
    return;
  }
  for (uint64_t r = gwarp; r < n; r += gwarps) {
    const uint32_t* q = p.enc + (b0 + r) * p.W;
    const int32_t y = p.labels[b0 + r];
    uint32_t best = 0, bestp = kFull, truep = 0;
    for (uint32_t c = 0; c < p.C; ++c) {
      const uint32_t* v = p.cv + static_cast<uint64_t>(c) * p.W;
      uint32_t a = 0;
      for (uint32_t w = lane; w < p.W; w += 32u) a += __popc(__ldg(q + w) ^ v[w]);
      a = __reduce_add_sync(kFull, a);
      if (a < bestp) {
        bestp = a;
        best = c;
      }
      if (static_cast<int32_t>(c) == y) truep = a;
    }
    if (lane == 0) {
      best_out[r] = (static_cast<unsigned long long>(bestp) << 32) | best;
      p.truep[r] = truep;
    }
  }
}

// C >= 32: CTA-tiled scan (hv_scan.cuh) over (32-row tile, 32-class block)
// items; per-row argmin merged across class blocks with a 64-bit atomicMin.
__device__ void score_tiled(const OnlineParams& p, unsigned long long* best_out, ScanSmem& s, uint64_t b0, uint32_t n,
                            uint32_t lane, uint32_t warp) {
  __shared__ int s_last;
  const uint32_t ncb = (p.C + kScanCls - 1) / kScanCls;
  const uint64_t ntiles = (n + kScanRows - 1) / kScanRows;
  const uint32_t ks = p.ksplit;
  for (uint64_t it = blockIdx.x; it < ntiles * ncb * ks; it += gridDim.x) {
    // a batch has few row tiles, so the word range is split across CTAs too;
    // the last of a tile's ks items to arrive owns the argmin
    const uint32_t kx = static_cast<uint32_t>(it % ks);
    const uint64_t tc = it / ks;
    const uint32_t cb = static_cast<uint32_t>(tc % ncb);
    const uint64_t t0 = (tc / ncb) * kScanRows;
    const uint32_t nr = static_cast<uint32_t>(min(static_cast<uint64_t>(kScanRows), n - t0));
    const uint32_t kbeg = static_cast<uint32_t>((static_cast<uint64_t>(p.W) * kx / ks) & ~3ull);
    const uint32_t kend = kx + 1 == ks ? p.W : static_cast<uint32_t>((static_cast<uint64_t>(p.W) * (kx + 1) / ks) & ~3ull);
    uint32_t a[kScanRowsPerWarp];
    const uint32_t c = cb * kScanCls + lane;
    const bool compute = warp < kScanRows / kScanRowsPerWarp;
    if (p.pre) {  // tensor-core popcounts of this batch (uniform per launch)
#pragma unroll
      for (int k = 0; k < kScanRowsPerWarp; ++k) {
        const uint32_t r = warp * kScanRowsPerWarp + k;
        a[k] = 0u;
        if (compute && r < nr && c < p.C) {
          uint32_t* slot = p.pre + (t0 + r) * p.C + c;
          a[k] = *slot;
          *slot = 0u;  // the next batch's split-K partials add into zeros
        }
      }
    } else {
      scan_tile<kOThreads>(p.enc, b0 + t0, nr, p.W, p.cv, p.C, cb * kScanCls, s, a, kbeg, kend);
    }
    if (ks > 1) {
      if (compute && c < p.C) {
#pragma unroll
        for (int k = 0; k < kScanRowsPerWarp; ++k) {
          const uint32_t r = warp * kScanRowsPerWarp + k;
          if (r < nr) atomicAdd(p.pscr + (t0 + r) * p.C + c, a[k]);
        }
      }
      __threadfence();
      __syncthreads();
      if (threadIdx.x == 0) s_last = atomicAdd(p.arrive + tc, 1u) == ks - 1;
      __syncthreads();
      if (!s_last) continue;  // uniform per CTA
      __threadfence();
      if (compute && c < p.C) {
#pragma unroll
        for (int k = 0; k < kScanRowsPerWarp; ++k) {
          const uint32_t r = warp * kScanRowsPerWarp + k;
          if (r < nr) {
            uint32_t* slot = p.pscr + (t0 + r) * p.C + c;
            a[k] = __ldcg(slot);
            *slot = 0u;  // zero for the next batch
          }
        }
      }
      if (threadIdx.x == 0) p.arrive[tc] = 0u;
    }
    if (compute) {
#pragma unroll
      for (int k = 0; k < kScanRowsPerWarp; ++k) {
        const uint32_t r = warp * kScanRowsPerWarp + k;
        if (r >= nr) break;
        const uint64_t row = t0 + r;
        const unsigned long long key = warp_min_u64(c < p.C ? scan_key(a[k], c) : ~0ull);
        if (lane == 0) atomicMin(best_out + row, key);
        if (c < p.C && static_cast<int32_t>(c) == p.labels[b0 + row]) p.truep[row] = a[k];
      }
    }
  }
}

// ------------------------------------------------------------- binarise ----
// Thread (warp ww, lane l) of a replay item owns bit l of words
// wb*8*COLS + ww + 8i, i < COLS. Stores its accumulators and, for touched classes, the re-binarised
// class words (model.cpp:139-163).
template <int COLS>
__device__ __forceinline__ void store_columns(const OnlineParams& p, uint32_t c, uint32_t wb, const double (&a)[COLS],
                                              double total, bool binarize) {
  const uint32_t lane = threadIdx.x & 31u, ww = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i < COLS; ++i) {
    const uint32_t w = wb * RTile<COLS>::kWords + ww + 8u * i;
    const uint32_t j = w * 32u + lane;
    const bool col = w < p.W && j < p.D;
    if (col) p.acc[static_cast<uint64_t>(c) * p.D + j] = a[i];
    if (binarize) {
      uint32_t bit = 0;
      if (col) {
        const double twice = 2.0 * a[i];
        bit = twice > total ? 1u : (twice < total ? 0u : ((p.tie[w] >> lane) & 1u));
      }
      const uint32_t word = __ballot_sync(kFull, bit);
      if (lane == 0 && w < p.W) p.cv[static_cast<uint64_t>(c) * p.W + w] = word;
    }
  }
}

template <int COLS>
__device__ __forceinline__ void load_columns(const OnlineParams& p, uint32_t c, uint32_t wb, double (&a)[COLS]) {
  const uint32_t lane = threadIdx.x & 31u, ww = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i < COLS; ++i) {
    const uint32_t w = wb * RTile<COLS>::kWords + ww + 8u * i;
    const uint32_t j = w * 32u + lane;
    a[i] = (w < p.W && j < p.D) ? p.acc[static_cast<uint64_t>(c) * p.D + j] : 0.0;
  }
}

// a[i] += v for the entries whose word (ww + 8i) has this lane's bit set, in
// entry order; branch-free: an unset bit adds +0.0, which leaves every
// accumulator bit-identical (acc is never -0.0: it starts from counts and
// x + y == 0 rounds to +0.0).
template <int COLS>
__device__ __forceinline__ void replay_chunk(const uint32_t* words, const double* val, uint32_t m, double (&a)[COLS]) {
  if constexpr (COLS == 1) {
    // word-major staging (word ww of rows k.. at ww * kWordPitch + k, see
    // staged_word): a warp reads 4 rows' words with one broadcast LDS.128
    // instead of one LDS per row — 8 warps x 1 wavefront per row was the
    // replay's shared-memory bill. Rows past m were staged as 0 words and
    // +0.0 values, so the loop runs in whole groups of 4.
    const uint32_t lane = threadIdx.x & 31u, ww = threadIdx.x >> 5;
    const uint32_t* wv = words + ww * kWordPitch;
    double acc = a[0];
#pragma unroll 8
    for (uint32_t k = 0; k < m; k += 4) {
      const uint4 w4 = *reinterpret_cast<const uint4*>(wv + k);
      const double2 v01 = *reinterpret_cast<const double2*>(val + k);
      const double2 v23 = *reinterpret_cast<const double2*>(val + k + 2);
      acc = __dadd_rn(acc, ((w4.x >> lane) & 1u) ? v01.x : 0.0);
      acc = __dadd_rn(acc, ((w4.y >> lane) & 1u) ? v01.y : 0.0);
      acc = __dadd_rn(acc, ((w4.z >> lane) & 1u) ? v23.x : 0.0);
      acc = __dadd_rn(acc, ((w4.w >> lane) & 1u) ? v23.y : 0.0);
    }
    a[0] = acc;
    return;
  }

  const uint32_t lane = threadIdx.x & 31u, ww = threadIdx.x >> 5;
  constexpr int kUnroll = COLS == 1 ? HV_REPLAY_UNROLL : 2;  // enough independent loads in flight ahead of the chain
#pragma unroll kUnroll
  for (uint32_t k = 0; k < m; ++k) {
    const double v = val[k];
#pragma unroll
    for (int i = 0; i < COLS; ++i) {
      const uint32_t wd = words[k * RTile<COLS>::kWords + ww + 8 * i];
      a[i] = __dadd_rn(a[i], ((wd >> lane) & 1u) ? v : 0.0);
    }
  }
}

struct Smem {
  uint32_t words[2][8 * kWordPitch];  // >= kOTile: COLS = 1 uses the padded word-major layout
  double val[2][kLChunk];
  uint8_t flag[2][kLChunk];  // MERGED: bit0 listed, bit1 true sample; lists: true sample
  uint32_t warpcnt[kLChunk / 32];
  uint32_t gmask[2][kLChunk / 32];  // MERGED (mw < 8): listed rows of each 32-row group of a chunk
  double weight;
  uint32_t dyn_item;
  uint16_t order[kOrderMax];  // LISTS + dynamic: classes by decreasing list length
};

// The class weight of class c over the batch's true samples, in sample order
// (model.cpp:268), and its sample count: threads 32.. stage the deltas of a
// 256-row chunk (+0.0 for other rows) while thread 0 runs the dependent chain
// over the previous one; then the result is published to the replay items
// through the class's epoch flag (release; the items acquire it).
// LISTS = true: walk the class's list (built by the list phase) instead of
// every row of the batch; its true entries carry their delta.
template <bool LISTS>
__device__ void class_weight_task(const OnlineParams& p, Smem& s, uint64_t b0, uint32_t n, uint32_t c,
                                  const double* w_in, double* w_out, uint32_t epoch) {
  const uint32_t tid = threadIdx.x;
  double wsum = *w_in;
  uint64_t ntrue = 0;
  if (LISTS) n = p.llen[c];
  auto fill = [&](uint32_t ch, uint32_t buf) {
    if (tid >= 32 && tid < 32 + kLChunk) {
      const uint32_t k = tid - 32, e = ch + k;
      bool is_t = false;
      double v = 0.0;
      if (e < n) {
        if (LISTS) {
          const uint32_t r = p.lidx[static_cast<uint64_t>(c) * p.bsz + e];
          is_t = p.labels[b0 + r] == static_cast<int32_t>(c);
          if (is_t) v = p.lval[static_cast<uint64_t>(c) * p.bsz + e];
        } else {
          is_t = p.labels[b0 + e] == static_cast<int32_t>(c);
          if (is_t) v = delta_of(p.truep[e], p.D);
        }
      }
      s.val[buf][k] = v;
      s.flag[buf][k] = is_t ? 1 : 0;
      // warps 1-8 cover one 32-entry group each (kLChunk = 256)
      const uint32_t gm = __ballot_sync(kFull, is_t);
      if ((tid & 31u) == 0) s.gmask[buf][k >> 5] = gm;
    }
  };
  fill(0, 0);
  __syncthreads();
  uint32_t buf = 0;
  for (uint32_t ch = 0; ch < n; ch += kLChunk, buf ^= 1u) {
    if (ch + kLChunk < n) fill(ch + kLChunk, buf ^ 1u);
    if (tid == 0) {
      const uint32_t m = min(static_cast<uint32_t>(kLChunk), n - ch);
      // per 32-entry group of true samples: none → skipped; a few → only their
      // adds (model.cpp adds δ for true samples only; the other entries are
      // +0.0); many → all 32, four per step (two LDS.128), 32 in flight, only
      // the adds serial. A rare class's weight chain is then a few adds
      // instead of a whole batch of +0.0 adds on its items' critical path.
      for (uint32_t g = 0; g * 32u < m; ++g) {
        uint32_t gm = s.gmask[buf][g];
        if (gm == 0u) continue;
        const double* vg = &s.val[buf][g * 32u];
        ntrue += __popc(gm);
        if (__popc(gm) > 8 && !(p.ablate & 256u)) {
#pragma unroll
          for (uint32_t k = 0; k < 32u; k += 4) {
            const double2 v01 = *reinterpret_cast<const double2*>(vg + k);
            const double2 v23 = *reinterpret_cast<const double2*>(vg + k + 2);
            wsum = __dadd_rn(wsum, v01.x);
            wsum = __dadd_rn(wsum, v01.y);
            wsum = __dadd_rn(wsum, v23.x);
            wsum = __dadd_rn(wsum, v23.y);
          }
        } else {
          while (gm != 0u) {
            wsum = __dadd_rn(wsum, vg[__ffs(gm) - 1]);
            gm &= gm - 1u;
          }
        }
      }
    }
    __syncthreads();
  }
  if (tid == 0) {
    *w_out = wsum;
    p.counts[c] += ntrue;
    __threadfence();
    st_release_u32(p.wflag + c, epoch);
  }
  __syncthreads();  // s reuse
}

__device__ __forceinline__ void await_class_weight(const OnlineParams& p, uint32_t c, uint32_t epoch) {
  const unsigned long long t0 = gtimer();
  while (ld_acquire_u32(p.wflag + c) != epoch) {
    if (gtimer() - t0 > 2000000000ull) __trap();  // 2 s: a lost task is a bug, never a hang
  }
}

// The next batch's rows into L2 during this batch's replay, so the next score
// phase reads them from L2 rather than HBM: thread t of `nthr` (over the
// participating CTAs) takes every nthr-th 128-byte line (CHB-MIT: score phase
// 4.1 -> 3.6 us per batch of 1,024).
__device__ __forceinline__ void prefetch_next_batch(const OnlineParams& p, uint64_t b0, uint64_t t, uint64_t nthr) {
  if (b0 + p.bsz >= p.rows || (p.ablate & 8u)) return;
  const uint64_t nrows = min(p.bsz, p.rows - (b0 + p.bsz));
  const char* base = reinterpret_cast<const char*>(p.enc + (b0 + p.bsz) * p.W);
  const uint64_t lines = (nrows * p.W * 4u + 127u) / 128u;
  for (uint64_t l = t; l < lines; l += nthr) asm volatile("prefetch.global.L2 [%0];" ::"l"(base + l * 128u));
}

// ------------------------------------------ MERGED replay, narrow items ----
// Items of MW = 4 words instead of 8, so the dense class's items spread over
// twice as many SMs, one replay warp per scheduler (a 1,024-row chain runs at
// ~11 cycles per row alone on its scheduler, ~15.5 with two warps per
// scheduler: scripts/probe_replay.cu). The CTA's other five warps stage the
// chunks — raw loads for chunk k+1 issued before chunk k's replay, flags and
// values (an fp64 division per true sample) formed after it — so the replay
// warps run nothing but their chains. A 32-row group with no listed row of the
// item's class is skipped (its adds would all be +0.0): with unbalanced
// classes (CHB-MIT: 0.3 % positives) the rare class's items replay a few
// groups; chunks with every group listed take the loop without the tests.
template <int MW>
__device__ void replay_merged_mw(const OnlineParams& p, const unsigned long long* bestv, Smem& s, uint64_t b0,
                                 uint32_t n, uint32_t par) {
  constexpr uint32_t kRows = kLChunk;  // rows per staged chunk
  constexpr uint32_t kThr = MW * 32;   // replay threads (warps 0 .. MW-1)
  constexpr uint32_t kStg = kOThreads - kThr;  // staging threads (the other warps)
  constexpr int kRowsPer = (kRows + kStg - 1) / kStg;
  constexpr int kLoads = (kRows * MW + kStg - 1) / kStg;
  static_assert(kRows + 4 <= kWordPitch && MW <= 8 && kStg % 32 == 0, "staging layout");
  const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
  const uint32_t st = tid - kThr;  // staging thread index (tid >= kThr)
  const uint32_t nwb = (p.W + MW - 1) / MW;
  const uint64_t items = static_cast<uint64_t>(p.C) * nwb;
  // separate weight tasks when every item has a CTA, or when the items past
  // the item CTAs are handed out dynamically
  const bool sep = p.wflag != nullptr && (gridDim.x >= items + p.C || (p.item_ctr != nullptr && gridDim.x > p.C));
  const uint32_t epoch = static_cast<uint32_t>(b0 / p.bsz) + 1u;
  if (sep && blockIdx.x < p.C) {
    const uint32_t c = blockIdx.x;
    class_weight_task<false>(p, s, b0, n, c, p.weight + par * p.C + c, p.weight + (par ^ 1u) * p.C + c, epoch);
  }
  const uint32_t first = sep ? p.C : 0u, stride = gridDim.x - first;
  // one CTA per SM (a second CTA on an SM halves both replays' rate): item
  // CTA k takes item k, and the items past the item CTAs go to whichever CTAs
  // finish first — with unbalanced classes the rare class's short items. Every
  // item CTA draws until it draws past the end, so the counter advances by
  // max(items, stride) per batch and batch bi's draws start at bi * that.
  const uint64_t dbase = static_cast<uint64_t>(b0 / p.bsz) * (items > stride ? items : stride);
  auto next_item = [&](uint64_t item) -> uint64_t {
    if (p.item_ctr == nullptr) return item + stride;
    if (tid == 0) s.dyn_item = atomicAdd(p.item_ctr, 1u);
    __syncthreads();
    const uint64_t d = static_cast<uint64_t>(s.dyn_item) - dbase + stride;
    __syncthreads();
    return d;
  };
  for (uint64_t item = blockIdx.x - first; blockIdx.x >= first; item = next_item(item)) {
    if (item >= items) {
      if (p.item_ctr == nullptr || item >= stride) break;  // a dynamic CTA without a first item still draws once
      continue;
    }
    const uint32_t c = static_cast<uint32_t>(item / nwb);
    const uint32_t wb = static_cast<uint32_t>(item % nwb);
    const uint32_t w = wb * MW + warp, j = w * 32u + lane;
    const bool col = tid < kThr && w < p.W && j < p.D;
    double acc = col ? p.acc[static_cast<uint64_t>(c) * p.D + j] : 0.0;
    double wsum = p.weight[par * p.C + c];
    uint64_t ntrue = 0;
    uint32_t mine = 0;  // this thread staged a listed row
    // staging thread st owns rows st + kStg * i of a chunk and words st + kStg * i
    bool rok[kRowsPer];
    int32_t ry[kRowsPer];
    unsigned long long rb[kRowsPer];
    uint32_t rt[kRowsPer];
    uint32_t rw[kLoads];
    auto load_chunk = [&](uint32_t ch) {  // raw loads only
#pragma unroll
      for (int i = 0; i < kRowsPer; ++i) {
        const uint32_t k = st + kStg * i;
        rok[i] = k < kRows && ch + k < n;
        if (rok[i]) {
          ry[i] = p.labels[b0 + ch + k];
          rb[i] = bestv[ch + k];
          rt[i] = p.truep[ch + k];
        }
      }
#pragma unroll
      for (int i = 0; i < kLoads; ++i) {
        const uint32_t e = st + i * kStg;
        const uint32_t k = e / MW, wl = e % MW;
        const uint32_t wg = wb * MW + wl;
        rw[i] = (k < kRows && ch + k < n && wg < p.W) ? __ldg(p.enc + (b0 + ch + k) * p.W + wg) : 0u;
      }
    };
    auto store_chunk = [&](uint32_t buf) {
#pragma unroll
      for (int i = 0; i < kRowsPer; ++i) {
        const uint32_t k = st + kStg * i;
        uint8_t rf = 0;
        double rv = 0.0;
        if (rok[i]) {
          const bool is_t = ry[i] == static_cast<int32_t>(c);
          const bool is_p = !is_t && static_cast<uint32_t>(rb[i]) == c;
          if (is_t) rv = delta_of(rt[i], p.D);
          if (is_p) rv = penalty_of(rb[i], p.gamma, p.D);
          rf = (is_t || is_p ? 1 : 0) | (is_t ? 2 : 0);
        }
        if (k < kRows) {
          s.val[buf][k] = rv;
          s.flag[buf][k] = rf;
        }
        mine |= rf & 1u;
        // rows k of one staging warp and one i are a 32-row group (kStg % 32 == 0)
        const uint32_t gm = __ballot_sync(kFull, rf & 1u);
        if (lane == 0 && k < kRows) s.gmask[buf][k >> 5] = gm;
      }
#pragma unroll
      for (int i = 0; i < kLoads; ++i) {
        const uint32_t e = st + i * kStg;
        const uint32_t k = e / MW, wl = e % MW;
        if (k < kRows) s.words[buf][wl * kWordPitch + k] = rw[i];
      }
    };
    // the next batch's rows into L2 (its score phase then reads them from L2,
    // not HBM): the staging warps of every item CTA take a slice, once per batch
    if (tid >= kThr && item == blockIdx.x - first) {
      prefetch_next_batch(p, b0, static_cast<uint64_t>(blockIdx.x - first) * kStg + (tid - kThr),
                          static_cast<uint64_t>(stride) * kStg);
    }
    const bool pr = p.prof != nullptr && blockIdx.x == ((p.ablate & 128u) ? gridDim.x - 1u : first) && tid == 0;
    const unsigned long long q0 = pr ? gtimer() : 0ull;
    // staging runs a chunk ahead of the replay and its raw loads two ahead:
    // chunk k + 2's loads are issued right after chunk k + 1 is stored, so an
    // L2 round trip hides behind a whole chunk's replay
    if (tid >= kThr) {
      load_chunk(0);
      store_chunk(0);
      if (kRows < n) load_chunk(kRows);
    }
    __syncthreads();
    const unsigned long long q1 = pr ? gtimer() : 0ull;
    uint32_t buf = 0;
    for (uint32_t ch = 0; ch < n; ch += kRows, buf ^= 1u) {
      const bool more = ch + kRows < n;
      const uint32_t m = min(kRows, n - ch);
      if (tid < kThr) {
        // rows past m were staged as 0 words and +0.0 values: whole groups of 32
        const uint32_t* wv = s.words[buf] + warp * kWordPitch;
        const double* val = s.val[buf];
        const uint32_t ng = (m + 31u) / 32u;
        auto group = [&](uint32_t g) {
#pragma unroll
          for (uint32_t k = g * 32u; k < g * 32u + 32u; k += 4) {
            const uint4 w4 = *reinterpret_cast<const uint4*>(wv + k);
            const double2 v01 = *reinterpret_cast<const double2*>(val + k);
            const double2 v23 = *reinterpret_cast<const double2*>(val + k + 2);
            acc = __dadd_rn(acc, ((w4.x >> lane) & 1u) ? v01.x : 0.0);
            acc = __dadd_rn(acc, ((w4.y >> lane) & 1u) ? v01.y : 0.0);
            acc = __dadd_rn(acc, ((w4.z >> lane) & 1u) ? v23.x : 0.0);
            acc = __dadd_rn(acc, ((w4.w >> lane) & 1u) ? v23.y : 0.0);
          }
        };
        bool dense = ng == kRows / 32u;
#pragma unroll
        for (uint32_t g = 0; g < kRows / 32u; ++g) dense = dense && s.gmask[buf][g] != 0u;
        if (dense) {
#pragma unroll 1
          for (uint32_t g = 0; g < kRows / 32u; g += 2) {  // no tests: 64 rows per iteration
            group(g);
            group(g + 1);
          }
        } else {
          for (uint32_t g = 0; g < ng; ++g) {
            if (s.gmask[buf][g] != 0u) group(g);  // warp-uniform
          }
        }
      } else {
        if (tid == kOThreads - 32 && !sep) {  // lane 0 of the last warp: the class weight chain
#pragma unroll 8
          for (uint32_t k = 0; k < m; ++k) {
            const uint8_t f = s.flag[buf][k];
            wsum = __dadd_rn(wsum, (f & 2u) ? s.val[buf][k] : 0.0);
            ntrue += f >> 1;
          }
        }
        if (more && !(p.ablate & 4u)) store_chunk(buf ^ 1u);  // the other buffer was last read before the previous barrier
        if (ch + 2u * kRows < n && !(p.ablate & 1u)) load_chunk(ch + 2u * kRows);
      }
      __syncthreads();
    }
    const unsigned long long q2 = pr ? gtimer() : 0ull;
    if (tid == kOThreads - 32) {
      if (sep) {
        await_class_weight(p, c, epoch);
        s.weight = p.weight[(par ^ 1u) * p.C + c];
      } else {
        s.weight = wsum;
      }
    }
    const int touched = __syncthreads_or(mine);
    const unsigned long long q3 = pr ? gtimer() : 0ull;
    if (tid < kThr) {
      // model.cpp:139-163: accumulators back, touched classes re-binarised
      if (col) p.acc[static_cast<uint64_t>(c) * p.D + j] = acc;
      if (touched) {
        uint32_t bit = 0;
        if (col) {
          const double twice = 2.0 * acc, total = s.weight;
          bit = twice > total ? 1u : (twice < total ? 0u : ((p.tie[w] >> lane) & 1u));
        }
        const uint32_t word = __ballot_sync(kFull, bit);
        if (lane == 0 && w < p.W) p.cv[static_cast<uint64_t>(c) * p.W + w] = word;
      }
    }
    if (pr) {
      p.prof[3] += q1 - q0;
      p.prof[4] += q2 - q1;
      p.prof[5] += q3 - q2;
      p.prof[6] += gtimer() - q3;
    }
    if (!sep && wb == 0 && tid == kOThreads - 32) {
      p.weight[(par ^ 1u) * p.C + c] = wsum;
      p.counts[c] += ntrue;
    }
    __syncthreads();  // s.weight reuse by the next item
  }
}

// ------------------------------------------------------- MERGED replay ----
template <int COLS>
__device__ void replay_merged(const OnlineParams& p, const unsigned long long* bestv, Smem& s, uint64_t b0, uint32_t n,
                              uint32_t par) {
  const uint32_t tid = threadIdx.x, lane = tid & 31u;
  const uint32_t nwb = (p.W + RTile<COLS>::kWords - 1) / RTile<COLS>::kWords;
  const uint64_t items = static_cast<uint64_t>(p.C) * nwb;
  // With spare CTAs, the class weights (a dependent chain over every true
  // sample of the batch) run as separate tasks on CTAs without a replay item
  // and publish through an epoch flag, instead of a weight warp inside every
  // item whose chain was on the item's critical path.
  const bool sep = p.wflag != nullptr && gridDim.x >= items + p.C;
  const uint32_t epoch = static_cast<uint32_t>(b0 / p.bsz) + 1u;
  if (sep && blockIdx.x >= items && blockIdx.x < items + p.C) {
    const uint32_t c = static_cast<uint32_t>(blockIdx.x - items);
    class_weight_task<false>(p, s, b0, n, c, p.weight + par * p.C + c, p.weight + (par ^ 1u) * p.C + c, epoch);
  }
  for (uint64_t item = blockIdx.x; item < items; item += gridDim.x) {
    const uint32_t c = static_cast<uint32_t>(item / nwb);
    const uint32_t wb = static_cast<uint32_t>(item % nwb);
    double a[COLS];
    if (tid < kOReplay) load_columns<COLS>(p, c, wb, a);
    double wsum = p.weight[par * p.C + c];
    uint64_t ntrue = 0;
    uint32_t mine = 0;  // this thread staged a listed row
    // registers holding the next chunk
    uint32_t rw[kLoadsPer];
    double rv = 0.0;
    uint8_t rf = 0;
    auto load_chunk = [&](uint32_t ch) {
      const uint32_t r = ch + tid;
      rf = 0;
      rv = 0.0;
      if (tid < RTile<COLS>::kChunk && r < n) {
        const int32_t y = p.labels[b0 + r];
        const unsigned long long bst = bestv[r];
        const bool is_t = y == static_cast<int32_t>(c);
        const bool is_p = !is_t && static_cast<uint32_t>(bst) == c;
        if (is_t) rv = delta_of(p.truep[r], p.D);
        if (is_p) rv = penalty_of(bst, p.gamma, p.D);
        rf = (is_t || is_p ? 1 : 0) | (is_t ? 2 : 0);
      }
#pragma unroll
      for (int i = 0; i < kLoadsPer; ++i) {
        const uint32_t e = tid + i * kOThreads;
        const uint32_t k = e / RTile<COLS>::kWords, ww = e % RTile<COLS>::kWords;
        const uint32_t w = wb * RTile<COLS>::kWords + ww;
        rw[i] = (k < RTile<COLS>::kChunk && ch + k < n && w < p.W) ? __ldg(p.enc + (b0 + ch + k) * p.W + w) : 0u;
      }
    };
    auto store_chunk = [&](uint32_t buf) {
      if (tid < RTile<COLS>::kChunk) {
        s.val[buf][tid] = rv;
        s.flag[buf][tid] = rf;
      }
      mine |= rf & 1u;
#pragma unroll
      for (int i = 0; i < kLoadsPer; ++i) {
        const uint32_t e = tid + i * kOThreads;
        const uint32_t k = e / RTile<COLS>::kWords, ww = e % RTile<COLS>::kWords;
        if (k < RTile<COLS>::kChunk) s.words[buf][staged_word<COLS>(k, ww)] = rw[i];
      }
    };
    const bool pr = p.prof != nullptr && blockIdx.x == 0 && tid == 0;
    const unsigned long long q0 = pr ? gtimer() : 0ull;
    load_chunk(0);
    store_chunk(0);
    __syncthreads();
    const unsigned long long q1 = pr ? gtimer() : 0ull;
    uint32_t buf = 0;
    for (uint32_t ch = 0; ch < n; ch += RTile<COLS>::kChunk, buf ^= 1u) {
      const bool more = ch + RTile<COLS>::kChunk < n;
      if (more && !(p.ablate & 1u)) load_chunk(ch + RTile<COLS>::kChunk);  // in flight during the replay below
      const uint32_t m = min(static_cast<uint32_t>(RTile<COLS>::kChunk), n - ch);
      if (p.ablate & 2u) {
      } else if (tid < kOReplay) {
        replay_chunk<COLS>(s.words[buf], s.val[buf], m, a);  // non-listed rows carry +0.0
      } else if (lane == 0 && !sep) {
#pragma unroll 8
        for (uint32_t k = 0; k < m; ++k) {
          const uint8_t f = s.flag[buf][k];
          wsum = __dadd_rn(wsum, (f & 2u) ? s.val[buf][k] : 0.0);
          ntrue += f >> 1;
        }
      }
      if (more && !(p.ablate & 4u)) store_chunk(buf ^ 1u);  // the other buffer was last read before the previous barrier
      __syncthreads();
    }
    const unsigned long long q2 = pr ? gtimer() : 0ull;
    if (tid == kOReplay) {
      if (sep) {  // the weight task of class c publishes the batch's final weight
        await_class_weight(p, c, epoch);
        s.weight = p.weight[(par ^ 1u) * p.C + c];
      } else {
        s.weight = wsum;
      }
    }
    const int touched = __syncthreads_or(mine);
    const unsigned long long q3 = pr ? gtimer() : 0ull;
    if (tid < kOReplay) store_columns<COLS>(p, c, wb, a, s.weight, touched != 0);
    if (pr) {
      p.prof[3] += q1 - q0;  // first chunk staged
      p.prof[4] += q2 - q1;  // chunk loop (replay)
      p.prof[5] += q3 - q2;  // weight wait
      p.prof[6] += gtimer() - q3;
    }
    if (!sep && wb == 0 && tid == kOReplay) {
      p.weight[(par ^ 1u) * p.C + c] = wsum;
      p.counts[c] += ntrue;
    }
    __syncthreads();  // s.weight reuse by the next item
  }
}

// -------------------------------------------------------- LISTS phases ----
__device__ void build_lists(const OnlineParams& p, const unsigned long long* bestv, Smem& s, uint64_t b0, uint32_t n,
                            bool sep) {
  const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
  for (uint32_t c = blockIdx.x; c < p.C; c += gridDim.x) {
    double wsum = p.weight[c];
    uint64_t ntrue = 0;
    uint32_t len = 0;
    // the next chunk's label / key / true-class popcount are loaded while this
    // chunk is compacted (the chunks were latency-bound on these loads)
    int32_t y_n = -1;
    unsigned long long b_n = 0;
    uint32_t t_n = 0;
    auto fetch = [&](uint32_t ch) {
      const uint32_t r = ch + tid;
      y_n = -1;
      if (tid < kLChunk && r < n) {
        y_n = p.labels[b0 + r];
        b_n = bestv[r];
        t_n = p.truep[r];
      }
    };
    fetch(0);
    for (uint32_t ch = 0; ch < n; ch += kLChunk) {
      const int32_t y = y_n;
      const unsigned long long bst = b_n;
      const uint32_t tp = t_n;
      if (ch + kLChunk < n) fetch(ch + kLChunk);
      bool is_t = false, is_p = false;
      double v = 0.0;
      const uint32_t r = ch + tid;
      if (tid < kLChunk && r < n) {
        is_t = y == static_cast<int32_t>(c);
        is_p = !is_t && static_cast<uint32_t>(bst) == c;
        if (is_t) v = delta_of(tp, p.D);
        if (is_p) v = penalty_of(bst, p.gamma, p.D);
      }
      const bool flag = is_t || is_p;
      const uint32_t bal = __ballot_sync(kFull, flag);
      if (warp < kLChunk / 32 && lane == 0) s.warpcnt[warp] = __popc(bal);
      __syncthreads();
      uint32_t m = 0, off = 0;
#pragma unroll
      for (int k = 0; k < kLChunk / 32; ++k) {
        off += (static_cast<uint32_t>(k) < warp) ? s.warpcnt[k] : 0u;
        m += s.warpcnt[k];
      }
      if (flag) {
        const uint32_t pos = off + __popc(bal & ((1u << lane) - 1u));
        s.val[0][pos] = v;
        s.flag[0][pos] = is_t ? 2 : 0;
        p.lidx[static_cast<uint64_t>(c) * p.bsz + len + pos] = r;
        p.lval[static_cast<uint64_t>(c) * p.bsz + len + pos] = v;
      }
      __syncthreads();
      if (tid == kOReplay && !sep) {  // class weight over the true samples, in sample order
#pragma unroll 8
        for (uint32_t k = 0; k < m; ++k) {
          const uint8_t f = s.flag[0][k];
          wsum = __dadd_rn(wsum, f ? s.val[0][k] : 0.0);
          ntrue += f >> 1;
        }
      }
      len += m;
      __syncthreads();
    }
    if (tid == kOReplay) {
      if (!sep) {
        p.weight[c] = wsum;
        p.counts[c] += ntrue;
      }
      p.llen[c] = len;
    }
  }
}

// The list phase with (class, 256-row chunk) work items instead of one CTA
// walking all chunks of a class (used when the class weights run as separate
// tasks): an item counts the class's listed rows of all earlier chunks (labels
// and argmin keys only, the loads of several chunks in flight), then compacts
// its own chunk at that offset — the same contiguous row-ordered lists, but
// the phase takes ~2 L2 round trips instead of one per chunk (UCI-HAR batch
// 8,192: 32 sequential chunks per class before).
__device__ void build_lists_par(const OnlineParams& p, const unsigned long long* bestv, Smem& s, uint64_t b0,
                                uint32_t n) {
  const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
  const uint32_t nch = (n + kLChunk - 1) / kLChunk;
  const uint64_t items = static_cast<uint64_t>(p.C) * nch;
  for (uint64_t item = blockIdx.x; item < items; item += gridDim.x) {
    const uint32_t c = static_cast<uint32_t>(item / nch), j = static_cast<uint32_t>(item % nch);
    // listed rows of class c in chunks [0, j): per-thread counts over whole chunks
    uint32_t pre = 0;
    if (tid < kLChunk) {
#pragma unroll 4
      for (uint32_t q = 0; q < j; ++q) {
        const uint32_t r = q * kLChunk + tid;  // < n: earlier chunks are full
        const int32_t y = p.labels[b0 + r];
        const uint32_t bc = static_cast<uint32_t>(bestv[r]);
        pre += (y == static_cast<int32_t>(c) || bc == c) ? 1u : 0u;
      }
    }
    // own chunk: flags and values
    const uint32_t r = j * kLChunk + tid;
    bool is_t = false, is_p = false;
    double v = 0.0;
    if (tid < kLChunk && r < n) {
      const int32_t y = p.labels[b0 + r];
      const unsigned long long bst = bestv[r];
      is_t = y == static_cast<int32_t>(c);
      is_p = !is_t && static_cast<uint32_t>(bst) == c;
      if (is_t) v = delta_of(p.truep[r], p.D);
      if (is_p) v = penalty_of(bst, p.gamma, p.D);
    }
    const bool flag = is_t || is_p;
    const uint32_t bal = __ballot_sync(kFull, flag);
    pre = __reduce_add_sync(kFull, pre);
    if (warp < kLChunk / 32 && lane == 0) {
      s.warpcnt[warp] = __popc(bal);
      s.gmask[0][warp] = pre;  // per-warp prefix counts (scratch)
    }
    __syncthreads();
    uint32_t base = 0, off = 0, m = 0;
#pragma unroll
    for (int k = 0; k < kLChunk / 32; ++k) {
      base += s.gmask[0][k];
      off += (static_cast<uint32_t>(k) < warp) ? s.warpcnt[k] : 0u;
      m += s.warpcnt[k];
    }
    if (flag) {
      const uint32_t pos = base + off + __popc(bal & ((1u << lane) - 1u));
      p.lidx[static_cast<uint64_t>(c) * p.bsz + pos] = r;
      p.lval[static_cast<uint64_t>(c) * p.bsz + pos] = v;
    }
    if (j + 1 == nch && tid == 0) p.llen[c] = base + m;
    __syncthreads();  // warpcnt / gmask reuse
  }
}

template <int COLS>
__device__ void replay_lists(const OnlineParams& p, Smem& s, uint64_t b0, uint32_t n, bool sep) {
  const uint32_t tid = threadIdx.x;
  const uint32_t nwb = (p.W + RTile<COLS>::kWords - 1) / RTile<COLS>::kWords;
  const uint64_t items = static_cast<uint64_t>(p.C) * nwb;
  const uint32_t epoch = static_cast<uint32_t>(b0 / p.bsz) + 1u;
  // every CTA's last warp: a slice of the next batch's rows into L2
  if (tid >= kOThreads - 32) {
    prefetch_next_batch(p, b0, static_cast<uint64_t>(blockIdx.x) * 32u + (tid - (kOThreads - 32)),
                        static_cast<uint64_t>(gridDim.x) * 32u);
  }
  if (sep && blockIdx.x >= items && blockIdx.x < items + p.C) {
    const uint32_t c = static_cast<uint32_t>(blockIdx.x - items);
    class_weight_task<true>(p, s, b0, n, c, p.weight + c, p.weight + c, epoch);  // LISTS: weights in place
  }
  // items are handed out dynamically when a counter is given: per-class list
  // lengths vary (a class can collect hundreds of mispredicted rows), so a
  // static round robin left CTAs with long lists as the batch's tail. The
  // counter advances by exactly items + gridDim.x per batch (every CTA draws
  // one index past the end), so batch bi's indices start at bi * that.
  const uint64_t base = static_cast<uint64_t>(b0 / p.bsz) * (items + gridDim.x);
  // longest lists first (their items are the long ones): every CTA ranks the
  // classes itself (C^2 / 32 compares per lane), no extra grid barrier
  const bool ordered = p.item_ctr != nullptr && p.C <= kOrderMax;
  if (ordered) {
    for (uint32_t c = tid; c < p.C; c += blockDim.x) {
      const uint32_t lc = p.llen[c];
      uint32_t rank = 0;
      for (uint32_t d = 0; d < p.C; ++d) {
        const uint32_t ld = p.llen[d];
        rank += (ld > lc || (ld == lc && d < c)) ? 1u : 0u;
      }
      s.order[rank] = static_cast<uint16_t>(c);
    }
    __syncthreads();
  }
  for (uint64_t item = blockIdx.x;; item += gridDim.x) {
    if (p.item_ctr) {
      if (tid == 0) s.dyn_item = static_cast<uint32_t>(atomicAdd(p.item_ctr, 1u) - base);
      __syncthreads();
      item = s.dyn_item;
      __syncthreads();
    }
    if (item >= items) break;
    const uint32_t c = ordered ? s.order[item / nwb] : static_cast<uint32_t>(item / nwb);
    const uint32_t len = p.llen[c];
    if (len == 0) continue;  // untouched class: acc and class vector unchanged
    const uint32_t wb = static_cast<uint32_t>(item % nwb);
    const bool pr = p.prof != nullptr && blockIdx.x == 0 && tid == 0;
    const unsigned long long q0 = pr ? gtimer() : 0ull;
    double a[COLS];
    if (tid < kOReplay) load_columns<COLS>(p, c, wb, a);
    const uint32_t* li = p.lidx + static_cast<uint64_t>(c) * p.bsz;
    const double* lv = p.lval + static_cast<uint64_t>(c) * p.bsz;
    uint32_t rw[kLoadsPer];
    uint32_t ri[kLoadsPer];  // list entries (row indices) of the next chunk's gathers, loaded a chunk ahead
    double rv = 0.0;
    auto load_idx = [&](uint32_t k0) {
      const uint32_t m = min(static_cast<uint32_t>(RTile<COLS>::kChunk), len - k0);
#pragma unroll
      for (int i = 0; i < kLoadsPer; ++i) {
        const uint32_t k = (tid + i * kOThreads) / RTile<COLS>::kWords;
        ri[i] = k < m ? li[k0 + k] : 0u;
      }
    };
    // the row gathers take their addresses from ri: the list-index round trip
    // is not in front of every chunk's loads (Large: ~180 list entries per
    // class, 6 chunks of 32 per item)
    auto load_chunk = [&](uint32_t k0) {
      const uint32_t m = min(static_cast<uint32_t>(RTile<COLS>::kChunk), len - k0);
      if (tid < m) rv = lv[k0 + tid];
#pragma unroll
      for (int i = 0; i < kLoadsPer; ++i) {
        const uint32_t e = tid + i * kOThreads;
        const uint32_t k = e / RTile<COLS>::kWords, ww = e % RTile<COLS>::kWords;
        const uint32_t w = wb * RTile<COLS>::kWords + ww;
        rw[i] = (k < m && w < p.W) ? __ldg(p.enc + (b0 + ri[i]) * p.W + w) : 0u;
      }
    };
    auto store_chunk = [&](uint32_t buf) {
      if (tid < RTile<COLS>::kChunk) s.val[buf][tid] = rv;
#pragma unroll
      for (int i = 0; i < kLoadsPer; ++i) {
        const uint32_t e = tid + i * kOThreads;
        const uint32_t k = e / RTile<COLS>::kWords, ww = e % RTile<COLS>::kWords;
        if (k < RTile<COLS>::kChunk) s.words[buf][staged_word<COLS>(k, ww)] = rw[i];
      }
    };
    load_idx(0);
    load_chunk(0);
    if (RTile<COLS>::kChunk < len) load_idx(RTile<COLS>::kChunk);
    store_chunk(0);
    __syncthreads();
    const unsigned long long q1 = pr ? gtimer() : 0ull;
    uint32_t buf = 0;
    for (uint32_t k0 = 0; k0 < len; k0 += RTile<COLS>::kChunk, buf ^= 1u) {
      const bool more = k0 + RTile<COLS>::kChunk < len;
      if (more) {
        load_chunk(k0 + RTile<COLS>::kChunk);
        if (k0 + 2u * RTile<COLS>::kChunk < len) load_idx(k0 + 2u * RTile<COLS>::kChunk);
      }
      const uint32_t m = min(static_cast<uint32_t>(RTile<COLS>::kChunk), len - k0);
      if (tid < kOReplay) replay_chunk<COLS>(s.words[buf], s.val[buf], m, a);
      if (more) store_chunk(buf ^ 1u);
      __syncthreads();
    }
    if (sep) {
      if (tid == kOReplay) {
        await_class_weight(p, c, epoch);
        s.weight = p.weight[c];
      }
      __syncthreads();
    }
    const unsigned long long q2 = pr ? gtimer() : 0ull;
    if (tid < kOReplay) store_columns<COLS>(p, c, wb, a, sep ? s.weight : p.weight[c], true);
    if (sep) __syncthreads();  // s.weight reuse by the next item
    if (pr) {
      p.prof[3] += q1 - q0;           // columns + first chunk staged
      p.prof[4] += q2 - q1;           // chunk loop (+ weight wait)
      p.prof[6] += gtimer() - q2;     // store
      p.prof[5] += 1;                 // items this CTA ran (reported x1e3 per batch)
    }
  }
}

union __align__(16) OnlineSmem {
  Smem replay;
  ScanSmem scan;  // used only between the batch-start and the next grid barrier
};

template <bool MERGED, int COLS>
__global__ void __launch_bounds__(kOThreads, 2) online_persistent_kernel(OnlineParams p) {
  cg::grid_group grid = cg::this_grid();
  __shared__ OnlineSmem u;
  Smem& s = u.replay;
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  const uint64_t gwarps = static_cast<uint64_t>(gridDim.x) * (kOThreads / 32);
  const uint64_t gwarp = static_cast<uint64_t>(blockIdx.x) * (kOThreads / 32) + warp;
  const bool lane_class = p.tiled != 0;
  uint32_t par = 0;
  const bool prof = p.prof != nullptr && blockIdx.x == 0 && threadIdx.x == 0;
  unsigned long long t0 = prof ? gtimer() : 0ull, t1 = 0, t2 = 0;
  for (uint64_t b0 = 0; b0 < p.rows; b0 += p.bsz, par ^= 1u) {
    const uint32_t n = static_cast<uint32_t>(min(p.bsz, p.rows - b0));
    // per-row argmin keys, double-buffered by batch parity: the atomicMin
    // targets of the next batch are reset while this batch still reads its own
    unsigned long long* bestv = p.best + par * p.bsz;
    if (lane_class) {
      score_tiled(p, bestv, u.scan, b0, n, lane, warp);
    } else {
      score_warp_per_row(p, bestv, b0, n, gwarp, gwarps, lane);
    }
    grid.sync();
    if (prof) t1 = gtimer();
    t2 = t1;
    if constexpr (MERGED) {
      // profile: every CTA's own replay work time (p.prof[7 + CTA])
      const unsigned long long r0 = p.prof != nullptr && threadIdx.x == 0 ? gtimer() : 0ull;
      if (p.mw == 4) {
        replay_merged_mw<4>(p, bestv, s, b0, n, par);
      } else {
        replay_merged<COLS>(p, bestv, s, b0, n, par);
      }
      if (p.prof != nullptr && threadIdx.x == 0) {
        p.prof[7 + blockIdx.x] += gtimer() - r0;
        uint32_t sm;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
        p.prof[7 + 2048 + blockIdx.x] = sm;
      }
    } else {
      const uint64_t litems = static_cast<uint64_t>(p.C) * ((p.W + RTile<COLS>::kWords - 1) / RTile<COLS>::kWords);
      const bool sep = p.wflag != nullptr && gridDim.x >= litems + p.C;
      // (class, chunk) items from 4 chunks per batch on (UCI-HAR batch 8,192:
      // 69.6 -> 60.1 us per batch; batch 256, one chunk: 2 % slower, so not there)
      if (sep && n >= 4u * kLChunk && !(p.ablate & 32u)) {
        build_lists_par(p, bestv, s, b0, n);
      } else {
        build_lists(p, bestv, s, b0, n, sep);
      }
      grid.sync();
      if (prof) t2 = gtimer();
      replay_lists<COLS>(p, s, b0, n, sep);
    }
    if (lane_class) {
      // one batch per launch with precomputed popcounts: reset this batch's own keys
      unsigned long long* nxt = p.pre ? bestv : p.best + (par ^ 1u) * p.bsz;
      const uint64_t gt = static_cast<uint64_t>(blockIdx.x) * kOThreads + threadIdx.x;
      for (uint64_t r = gt; r < p.bsz; r += static_cast<uint64_t>(gridDim.x) * kOThreads) nxt[r] = ~0ull;
    }
    grid.sync();
    if (prof) {
      const unsigned long long t3 = gtimer();
      p.prof[0] += t1 - t0;
      p.prof[1] += t2 - t1;
      p.prof[2] += t3 - t2;
      t0 = t3;
    }
  }
}

// ---------------------------------------------------- small batches ----
// Small batches (the UCI-HAR batch sweep down to one sample): the persistent
// kernel's grid barriers (~3 us each, two per batch) dominate there. One
// thread-block cluster of kClCTAs CTAs runs every batch instead, with one
// cluster barrier per batch. CTA q owns a slice of the words, i.e. of the
// accumulator columns and class-vector words, and keeps both slices resident
// in shared memory for the whole run (written back once at the end):
//   1. the batch rows' slice is already staged (cp.async, issued during the
//      previous batch); partial Hamming popcounts of every (row, class) pair
//      over the slice are added into every CTA's totals through distributed
//      shared memory (batch-parity double buffer);
//   2. cluster barrier; every CTA derives the same predictions and add values
//      (model.cpp:259-276), per-class row lists in sample order, and class
//      weights / counts in that order;
//   3. every touched class: each thread replays the list on its elements of
//      the slice (independent chains, sample order per element) and
//      re-binarises them with the batch's final weight (model.cpp:139-163).
// Bit-identical to the reference like every other mode.
constexpr uint32_t kClCTAs = 8, kClThreads = 1024, kClMaxRows = 64, kClMaxC = 32, kClR = 4;
constexpr size_t kClDefaultRows = 16;  // measured crossover with the persistent kernel

__global__ void __cluster_dims__(kClCTAs, 1, 1) __launch_bounds__(kClThreads, 1)
    online_cluster_kernel(OnlineParams p) {
  cg::cluster_group cluster = cg::this_cluster();
  // dynamic: accs (C x ws*32 doubles) | xs (2 x nmax x ws words) | cvs (C x ws words)
  extern __shared__ __align__(16) uint8_t dyn[];
  __shared__ uint32_t tot[2][kClMaxRows][kClMaxC];
  __shared__ double vt[kClMaxRows], vp[kClMaxRows], wsm[kClMaxC];
  __shared__ int32_t ct[kClMaxRows], cp[kClMaxRows];
  __shared__ uint8_t lrow[kClMaxC][kClMaxRows];
  __shared__ double lv[kClMaxC][kClMaxRows];
  __shared__ uint32_t llen[kClMaxC];
  __shared__ unsigned long long cnt[kClMaxC];
  const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
  const uint32_t q = cluster.block_rank();
  const uint32_t W = p.W, C = p.C, D = p.D;
  const uint32_t ws = (W + kClCTAs - 1) / kClCTAs;  // words per CTA
  const uint32_t w0 = min(W, q * ws), w1 = min(W, w0 + ws), nw = w1 - w0;
  const uint32_t nmax = static_cast<uint32_t>(p.bsz);
  const uint32_t E = ws * 32u;  // accumulator elements per class in the slice
  double* accs = reinterpret_cast<double*>(dyn);
  uint32_t* xsb = reinterpret_cast<uint32_t*>(accs + static_cast<size_t>(C) * E);
  uint32_t* cvs = xsb + 2 * nmax * ws;
  for (uint32_t k = tid; k < C * E; k += kClThreads) {
    const uint32_t c = k / E, e = k % E, j = w0 * 32u + e;
    accs[k] = (e < nw * 32u && j < D) ? p.acc[static_cast<uint64_t>(c) * D + j] : 0.0;
  }
  for (uint32_t k = tid; k < C * nw; k += kClThreads) cvs[(k / nw) * ws + k % nw] = p.cv[(k / nw) * W + w0 + k % nw];
  for (uint32_t k = tid; k < 2 * kClMaxRows * kClMaxC; k += kClThreads) (&tot[0][0][0])[k] = 0;
  if (tid < C) {
    wsm[tid] = p.weight[tid];
    cnt[tid] = p.counts[tid];
  }
  auto stage = [&](uint64_t b, uint32_t buf) {  // rows [b, b + n) of the slice, asynchronously
    const uint32_t n = static_cast<uint32_t>(min(p.bsz, p.rows - b));
    uint32_t* xs = xsb + buf * nmax * ws;
    for (uint32_t k = tid; k < n * nw; k += kClThreads) {
      __pipeline_memcpy_async(xs + (k / nw) * ws + k % nw, p.enc + (b + k / nw) * W + w0 + k % nw, 4);
    }
    __pipeline_commit();
  };
  stage(0, 0);
  cluster.sync();  // every CTA's totals are zero before anyone adds
  uint32_t par = 0;
  for (uint64_t b0 = 0; b0 < p.rows; b0 += p.bsz, par ^= 1u) {
    const uint32_t n = static_cast<uint32_t>(min(p.bsz, p.rows - b0));
    const uint32_t* xs = xsb + par * nmax * ws;
    __pipeline_wait_prior(0);
    __syncthreads();
    if (b0 + p.bsz < p.rows) stage(b0 + p.bsz, par ^ 1u);  // lands during this batch
    for (uint32_t pr = warp; pr < n * C; pr += kClThreads / 32) {
      const uint32_t r = pr / C, c = pr % C;
      uint32_t a = 0;
      for (uint32_t w = lane; w < nw; w += 32) a += __popc(xs[r * ws + w] ^ cvs[c * ws + w]);
      a = __reduce_add_sync(kFull, a);
      if (lane < kClCTAs && a) atomicAdd(cluster.map_shared_rank(&tot[par][r][c], lane), a);
    }
    cluster.sync();
    if (tid < n) {  // pick_label (strict <, lowest class on ties), score_to_delta
      const int32_t y = p.labels[b0 + tid];
      uint32_t best = tot[par][tid][0], bc = 0;
      for (uint32_t c = 1; c < C; ++c) {
        if (tot[par][tid][c] < best) {
          best = tot[par][tid][c];
          bc = c;
        }
      }
      ct[tid] = y;
      vt[tid] = delta_of(tot[par][tid][y], D);
      const bool wrong = static_cast<int32_t>(bc) != y;
      cp[tid] = wrong ? static_cast<int32_t>(bc) : -1;
      vp[tid] = wrong ? penalty_of((static_cast<unsigned long long>(best) << 32) | bc, p.gamma, D) : 0.0;
    }
    __syncthreads();
    if (tid < C) {  // class tid: its rows in sample order; weight and count over its true samples
      uint32_t m = 0;
      double wsum = wsm[tid];
      for (uint32_t r = 0; r < n; ++r) {
        if (ct[r] == static_cast<int32_t>(tid)) {
          lrow[tid][m] = static_cast<uint8_t>(r);
          lv[tid][m++] = vt[r];
          wsum = __dadd_rn(wsum, vt[r]);
          cnt[tid] += 1;
        } else if (cp[r] == static_cast<int32_t>(tid)) {
          lrow[tid][m] = static_cast<uint8_t>(r);
          lv[tid][m++] = vp[r];
        }
      }
      llen[tid] = m;
      wsm[tid] = wsum;
    } else if (tid >= 64) {  // this batch's totals are consumed: zero them for batch b + 2
      for (uint32_t k = tid - 64; k < n * kClMaxC; k += kClThreads - 64) (&tot[par][0][0])[k] = 0;
    }
    __syncthreads();
    const uint32_t R = (nw * 32u + kClThreads - 1) / kClThreads;
    for (uint32_t c = 0; c < C; ++c) {
      const uint32_t m = llen[c];
      if (m == 0) continue;  // untouched: not re-binarised (uniform)
      double* ac = accs + static_cast<size_t>(c) * E;
      double a[kClR];
#pragma unroll
      for (uint32_t k = 0; k < kClR; ++k) a[k] = (k < R && k * (kClThreads / 32) + warp < nw) ? ac[k * kClThreads + tid] : 0.0;
      for (uint32_t e = 0; e < m; ++e) {
        const uint32_t* x = xs + lrow[c][e] * ws;
        const double v = lv[c][e];
#pragma unroll
        for (uint32_t k = 0; k < kClR; ++k) {
          const uint32_t w = k * (kClThreads / 32) + warp;  // local word
          if (k < R && w < nw && ((x[w] >> lane) & 1u)) a[k] = __dadd_rn(a[k], v);
        }
      }
      const double total = wsm[c];
#pragma unroll
      for (uint32_t k = 0; k < kClR; ++k) {
        if (k >= R) break;
        const uint32_t w = k * (kClThreads / 32) + warp, j = (w0 + w) * 32u + lane;
        uint32_t bit = 0;
        if (w < nw && j < D) {
          ac[k * kClThreads + tid] = a[k];
          const double twice = 2.0 * a[k];
          bit = twice > total ? 1u : (twice < total ? 0u : ((p.tie[w0 + w] >> lane) & 1u));
        }
        const uint32_t word = __ballot_sync(kFull, bit);
        if (lane == 0 && w < nw) cvs[c * ws + w] = word;
      }
    }
  }
  __syncthreads();
  for (uint32_t k = tid; k < C * E; k += kClThreads) {
    const uint32_t c = k / E, e = k % E, j = w0 * 32u + e;
    if (e < nw * 32u && j < D) p.acc[static_cast<uint64_t>(c) * D + j] = accs[k];
  }
  for (uint32_t k = tid; k < C * nw; k += kClThreads) p.cv[(k / nw) * W + w0 + k % nw] = cvs[(k / nw) * ws + k % nw];
  if (q == 0 && tid < C) {
    p.weight[tid] = wsm[tid];
    p.counts[tid] = cnt[tid];
  }
  cluster.sync();  // no CTA leaves while a peer may still add into its shared memory
}

__global__ void weight_copy_kernel(const double* __restrict__ src, double* __restrict__ dst, uint32_t C) {
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < C) dst[c] = src[c];
}

template <bool MERGED, int COLS>
unsigned cooperative_grid(hv_context* ctx, uint64_t want) {
  int per_sm = 0;
  ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, online_persistent_kernel<MERGED, COLS>, kOThreads, 0),
     "occupancy");
  if (per_sm < 1) fail(HV_ERR_CUDA, "online_persistent_kernel does not fit on an SM");
  uint64_t cap = static_cast<uint64_t>(ctx->sm_count) * static_cast<uint64_t>(per_sm);
  if (const char* g = getenv("HVB200_ONLINE_GRID")) cap = std::min<uint64_t>(cap, std::max(1, atoi(g)));
  return static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>(want, cap)));
}

}  // namespace

// All online batches over rows [0, rows) of `enc` (the bootstrap has already
// initialised acc/weight/counts/cv from the first batch's classical counts).
void train_online_persistent(hv_context* ctx, cudaStream_t st, const uint32_t* enc, size_t rows, size_t D,
                             const int32_t* labels, size_t C, size_t bsz, double gamma, const uint32_t* tie,
                             double* acc, double* weight, uint64_t* counts, uint32_t* cv) {
  if (rows == 0) return;
  const size_t W = words_per_row(D);
  const size_t n = std::min(bsz, rows);
  // small batches: one cluster, no grid barriers (HVB200_ONLINE_CLUSTER=0 disables, =N sets the row limit)
  const char* cl_env = getenv("HVB200_ONLINE_CLUSTER");
  const size_t cl_rows = cl_env ? static_cast<size_t>(atoi(cl_env)) : kClDefaultRows;
  const size_t ws = (W + kClCTAs - 1) / kClCTAs;
  const size_t cl_smem = C * ws * 32 * sizeof(double) + (2 * n + C) * ws * sizeof(uint32_t);
  if (n <= std::min<size_t>(cl_rows, kClMaxRows) && C <= kClMaxC && ws * 32 <= kClR * kClThreads &&
      cl_smem <= (180u << 10)) {
    OnlineParams p{};
    p.enc = enc;
    p.labels = labels;
    p.rows = rows;
    p.D = static_cast<uint32_t>(D);
    p.W = static_cast<uint32_t>(W);
    p.C = static_cast<uint32_t>(C);
    p.bsz = n;
    p.gamma = gamma;
    p.tie = tie;
    p.acc = acc;
    p.weight = weight;
    p.counts = counts;
    p.cv = cv;
    ck(cudaFuncSetAttribute(online_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            static_cast<int>(cl_smem)),
       "cudaFuncSetAttribute");
    online_cluster_kernel<<<kClCTAs, kClThreads, cl_smem, st>>>(p);
    launched("online_cluster_kernel");
    return;
  }
  // MERGED also for tiny batches: streaming a few rows per item is cheaper
  // than the extra grid barrier of the list phase
  const bool merged = C <= kMergedMaxC || n <= 32;
  uint32_t min_c = kLaneClassMinC;
  if (const char* e = getenv("HVB200_ONLINE_TILED_MIN_C")) min_c = static_cast<uint32_t>(atoi(e));
  const bool lane_class = C >= min_c;
  DevBuf<double> wts(2 * C, st), lval(merged ? 0 : C * n, st);
  DevBuf<unsigned long long> best(2 * n, st);
  DevBuf<uint32_t> truep(n, st), lidx(merged ? 0 : C * n, st), llen(merged ? 0 : C, st);
  weight_copy_kernel<<<grid_for(C, 128), 128, 0, st>>>(weight, wts.ptr, static_cast<uint32_t>(C));
  launched("weight_copy_kernel");
  if (lane_class) ck(cudaMemsetAsync(best.ptr, 0xFF, 2 * n * sizeof(unsigned long long), st), "memset");
  // long per-class lists (few classes): one chain per thread; short ones: four
  const bool cols4 = !merged && n < 64 * C;
  const bool cols8 = cols4 && n < 16 * C;
  // MERGED: 4-word items (replay_merged_mw; HVB200_ONLINE_MW=8 restores 8)
  uint32_t mw = 4;
  if (const char* e = getenv("HVB200_ONLINE_MW")) mw = atoi(e) == 8 ? 8u : 4u;
  const uint64_t iw = merged ? mw : cols8 ? 64 : cols4 ? 32 : 8;  // words per replay item
  const uint64_t items = static_cast<uint64_t>(C) * ((W + iw - 1) / iw);
  const uint64_t score_ctas = (n + kOThreads / 32 - 1) / (kOThreads / 32);
  // one extra CTA per class for the separate weight tasks
  const uint64_t want = std::max<uint64_t>(items + C, score_ctas);
  const char* wt_env = getenv("HVB200_ONLINE_WTASK");  // =0: class weights inside the items / list phase
  const bool wtask = !(wt_env && wt_env[0] == '0');
  DevBuf<uint32_t> wflag(wtask ? C : 0, st);
  if (wtask) wflag.zero();
  OnlineParams p{enc,     labels,   rows,     static_cast<uint32_t>(D), static_cast<uint32_t>(W),
                 static_cast<uint32_t>(C), n, gamma, tie, acc, wts.ptr, counts, cv, best.ptr, truep.ptr, lidx.ptr,
                 lval.ptr, llen.ptr, nullptr, lane_class ? 1u : 0u, 1u, nullptr, nullptr, nullptr, wtask ? wflag.ptr : nullptr,
                 nullptr, 0u, mw};
  DevBuf<uint32_t> item_ctr(merged ? 0 : 1, st);
  if (const char* ab = getenv("HVB200_ONLINE_ABLATE")) p.ablate = static_cast<uint32_t>(atoi(ab));  // timing only
  // HVB200_ONLINE_PROFILE=1: print the time per phase (CTA 0's view, barrier waits included)
  const char* pe = getenv("HVB200_ONLINE_PROFILE");
  DevBuf<unsigned long long> prof(pe && pe[0] == '1' ? 7 + 4096 : 0, st);
  if (prof.ptr) {
    prof.zero();
    p.prof = prof.ptr;
  }
  void* args[] = {&p};
  // tiled scoring: split the words so every CTA has a score item
  DevBuf<uint32_t> pscr, arrive;
  unsigned grid_est = 0;
  if (merged) {
    // narrow items, batches of >= 1,024 rows: at most one CTA per SM. A
    // cooperative grid larger than the SM count doubles up its lowest-numbered
    // CTAs (blocks 0-11 on six SMs for 160 CTAs, measured) and two replays on
    // one SM each run at ~2/3 of the rate; the items past the item CTAs are
    // handed out dynamically (CHB-MIT batch 1,024: 18.3 -> 17.7 us, batch
    // 8,192: 100.7 -> 80.9 us). Shorter batches keep every item on its own CTA
    // (batch 256: 9.9 vs 11.0 us: one chunk per item, a second item doubles it).
    const char* dyn = getenv("HVB200_ONLINE_DYNAMIC");  // =0: every item its own CTA, SMs doubled up (A/B)
    const bool dyn_ok = !(dyn && dyn[0] == '0') && n >= 4u * kLChunk;
    grid_est = cooperative_grid<true, 1>(ctx, mw == 4 && dyn_ok ? std::min<uint64_t>(want, ctx->sm_count) : want);
    const uint64_t draws = ((rows + n - 1) / n) * std::max<uint64_t>(items, grid_est);  // 32-bit counter
    if (mw == 4 && items + C > grid_est && draws < (1ull << 32) && dyn_ok) {
      item_ctr = DevBuf<uint32_t>(1, st);
      item_ctr.zero();
      p.item_ctr = item_ctr.ptr;
    }
  } else if (cols8) {
    grid_est = cooperative_grid<false, 8>(ctx, want);
  } else if (cols4) {
    grid_est = cooperative_grid<false, 4>(ctx, want);
  } else {
    grid_est = cooperative_grid<false, 1>(ctx, want);
  }
  // more replay items than CTAs (many classes, e.g. Large: 1,600 items on 296
  // CTAs): hand them out dynamically, longest lists first (replay 61.8 -> 47.3
  // us per batch at C = 100, D = 32768); with at most one item per CTA the
  // static assignment is already ideal
  if (!merged && items > grid_est) {
    item_ctr.zero();
    const char* dyn = getenv("HVB200_ONLINE_DYNAMIC");  // =0: static round robin (A/B)
    if (!(dyn && dyn[0] == '0')) p.item_ctr = item_ctr.ptr;
  }
  // many classes: score each batch on the tensor cores (hv_predict_tc.cu) and
  // run the persistent kernel once per batch on the precomputed popcounts
  const char* te = getenv("HVB200_ONLINE_TC");
  const bool tc_mode = !merged && lane_class && C >= 64 && (te == nullptr || te[0] != '0') && tc_usable(enc, D) &&
                       (n * W) % 4 == 0;
  if (lane_class && !tc_mode) {
    const uint64_t tiles = ((n + kScanRows - 1) / kScanRows) * ((C + kScanCls - 1) / kScanCls);
    // ~3 items per CTA keeps the tail of the score phase short
    const uint64_t ks = std::min<uint64_t>((3 * grid_est + tiles - 1) / tiles, std::max<size_t>(1, W / kScanK));
    if (ks > 1) {
      p.ksplit = static_cast<uint32_t>(ks);
      pscr = DevBuf<uint32_t>(n * C, st);
      arrive = DevBuf<uint32_t>(tiles, st);
      pscr.zero();
      arrive.zero();
      p.pscr = pscr.ptr;
      p.arrive = arrive.ptr;
    }
  }
  auto launch = [&](auto kern, unsigned grid) {
    ck(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(kern), dim3(grid), dim3(kOThreads), args, 0, st),
       "online_persistent_kernel");
  };
  if (tc_mode) {
    p.wflag = nullptr;  // one launch per batch restarts the epochs: weights stay in the list phase
    DevBuf<uint32_t> pre(n * C, st), cpop(C, st);
    DevBuf<uint8_t> img(tc_image_bytes(C, D), st);
    pre.zero();
    p.pre = pre.ptr;
    const auto kern = cols8 ? online_persistent_kernel<false, 8>
                            : cols4 ? online_persistent_kernel<false, 4> : online_persistent_kernel<false, 1>;
    for (size_t b0 = 0; b0 < rows; b0 += n) {
      const size_t nn = std::min(n, rows - b0);
      popc_tc_split(ctx, st, cv, C, D, enc + b0 * W, nn, cpop.ptr, pre.ptr, img.ptr);
      p.enc = enc + b0 * W;
      p.labels = labels + b0;
      p.rows = nn;
      if (p.item_ctr) ck(cudaMemsetAsync(p.item_ctr, 0, sizeof(uint32_t), st), "item counter");  // batch 0 of this launch
      launch(kern, grid_est);  // parity 0 only: best[0, n) was reset by the previous launch
    }
  } else if (merged) {
    launch(online_persistent_kernel<true, 1>, grid_est);
  } else if (cols8) {
    launch(online_persistent_kernel<false, 8>, cooperative_grid<false, 8>(ctx, want));
  } else if (cols4) {
    launch(online_persistent_kernel<false, 4>, cooperative_grid<false, 4>(ctx, want));
  } else {
    launch(online_persistent_kernel<false, 1>, cooperative_grid<false, 1>(ctx, want));
  }
  launched("online_persistent_kernel");
  if (prof.ptr) {
    unsigned long long h[7];
    ck(cudaMemcpyAsync(h, prof.ptr, sizeof(h), cudaMemcpyDeviceToHost, st), "D2H");
    ck(cudaStreamSynchronize(st), "sync");
    const double nb = static_cast<double>((rows + n - 1) / n);
    fprintf(stderr, "online phases (us/batch, %s, %d cols, ksplit %u): score %.2f lists %.2f replay %.2f"
            " [CTA 0 item: stage %.2f chunks %.2f weight-wait %.2f store %.2f]\n",
            merged ? "merged" : "lists", cols8 ? 8 : cols4 ? 4 : 1, p.ksplit, h[0] / nb / 1e3, h[1] / nb / 1e3,
            h[2] / nb / 1e3, h[3] / nb / 1e3, h[4] / nb / 1e3, h[5] / nb / 1e3, h[6] / nb / 1e3);
    if (merged) {  // the slowest CTAs' own replay work (weight tasks are CTAs 0 .. C-1 when separate)
      const unsigned g = grid_est;
      std::vector<unsigned long long> ct(g);
      ck(cudaMemcpy(ct.data(), prof.ptr + 7, g * sizeof(unsigned long long), cudaMemcpyDeviceToHost), "D2H");
      std::vector<unsigned> ord(g);
      for (unsigned i = 0; i < g; ++i) ord[i] = i;
      std::sort(ord.begin(), ord.end(), [&](unsigned a, unsigned b) { return ct[a] > ct[b]; });
      std::vector<unsigned long long> smv(g);
      ck(cudaMemcpy(smv.data(), prof.ptr + 7 + 2048, g * sizeof(unsigned long long), cudaMemcpyDeviceToHost), "D2H");
      std::vector<int> per(1024, 0);
      for (unsigned i = 0; i < g; ++i) per[smv[i] & 1023]++;
      int shared = 0;
      for (int v : per) shared += v > 1 ? v : 0;
      fprintf(stderr, "online replay: %d of %u CTAs share an SM; work per CTA (us/batch), slowest:", shared, g);
      for (unsigned i = 0; i < std::min(g, 10u); ++i)
        fprintf(stderr, " %u(sm%llu,%d):%.2f", ord[i], smv[ord[i]], per[smv[ord[i]] & 1023], ct[ord[i]] / nb / 1e3);
      fprintf(stderr, " | CTA 0: %.2f, CTA 1: %.2f, median %.2f\n", ct[0] / nb / 1e3, g > 1 ? ct[1] / nb / 1e3 : 0.0,
              ct[ord[g / 2]] / nb / 1e3);
    }
    if (!merged) {  // the last batch's per-class list lengths
      std::vector<uint32_t> len(C);
      ck(cudaMemcpy(len.data(), llen.ptr, C * sizeof(uint32_t), cudaMemcpyDeviceToHost), "D2H llen");
      uint64_t sum = 0, mx = 0;
      for (uint32_t v : len) {
        sum += v;
        mx = std::max<uint64_t>(mx, v);
      }
      fprintf(stderr, "online lists (last batch): mean %.1f max %llu entries per class; grid %u CTAs, %llu items\n",
              double(sum) / C, static_cast<unsigned long long>(mx), grid_est, static_cast<unsigned long long>(items));
    }
  }
  // MERGED leaves the final weights in the parity row after the last batch
  const size_t nb = (rows + n - 1) / n;
  const double* fin = merged ? wts.ptr + (nb & 1) * C : wts.ptr;
  weight_copy_kernel<<<grid_for(C, 128), 128, 0, st>>>(fin, weight, static_cast<uint32_t>(C));
  launched("weight_copy_kernel");
}

}  // namespace hvb
