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
//         C < 32: warp per row, lanes over words. C >= 32: lane = class over a
//         transposed copy of the class vectors (coalesced), 4 rows per warp,
//         per-row argmin merged across class blocks with a 64-bit atomicMin.
//
// Two classes (C <= kMergedMaxC) — MERGED:
//   replay  item = (class c, 8-word block): the batch is streamed in 256-row
//           chunks; each chunk's labels/scores and the 8 words of every row
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
//   replay  item = (class, 8-word block) over its own list only (classes
//           untouched by the batch are skipped), chunks prefetched as above.
//
// Touched classes are re-binarised with the batch's final weight
// (model.cpp:139-163, 277-279).
#include <cooperative_groups.h>

#include <algorithm>

#include "hv_internal.cuh"

namespace cg = cooperative_groups;

namespace hvb {
namespace {

constexpr uint32_t kFull = 0xFFFFFFFFu;
constexpr int kOWords = 8;                  // words per replay item
constexpr int kOChunk = 256;                // rows (MERGED) / list entries (LISTS) per chunk
constexpr int kOReplay = kOWords * 32;      // replay threads: one per bit column
constexpr int kOThreads = kOReplay + 32;    // + one warp for the weight chain
constexpr int kLoadsPer = (kOChunk * kOWords + kOThreads - 1) / kOThreads;  // word loads per thread per chunk
constexpr uint32_t kMergedMaxC = 2;  // more classes: per-class lists skip the other classes' rows
constexpr uint32_t kLaneClassMinC = 32;

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
  uint32_t* cvt;               // W x C transposed class vectors (lane-class scoring)
  unsigned long long* best;    // bsz: popc << 32 | class
  uint32_t* truep;             // bsz
  uint32_t* lidx;              // C x bsz (LISTS)
  double* lval;                // C x bsz (LISTS)
  uint32_t* llen;              // C (LISTS)
};

__device__ __forceinline__ double delta_of(uint32_t popc, uint32_t D) {
  return static_cast<double>(popc) / static_cast<double>(D);  // model.cpp:69-79 (IEEE division)
}

__device__ __forceinline__ double penalty_of(unsigned long long best, double gamma, uint32_t D) {
  return __dmul_rn(-gamma, __dsub_rn(1.0, delta_of(static_cast<uint32_t>(best >> 32), D)));
}

// ---------------------------------------------------------------- score ----
__device__ void score_warp_per_row(const OnlineParams& p, uint64_t b0, uint32_t n, uint64_t gwarp, uint64_t gwarps,
                                   uint32_t lane) {
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
      p.best[r] = (static_cast<unsigned long long>(bestp) << 32) | best;
      p.truep[r] = truep;
    }
  }
}

constexpr int kLcRows = 4;

__device__ void score_lane_class(const OnlineParams& p, uint64_t b0, uint32_t n, uint64_t gwarp, uint64_t gwarps,
                                 uint32_t lane) {
  const uint32_t ncb = (p.C + 31) / 32;
  const uint64_t ngr = (n + kLcRows - 1) / kLcRows;
  for (uint64_t it = gwarp; it < ngr * ncb; it += gwarps) {
    const uint32_t cb = static_cast<uint32_t>(it % ncb);
    const uint64_t r0 = (it / ncb) * kLcRows;
    const uint32_t c = cb * 32 + lane;
    const bool cok = c < p.C;
    const uint32_t* q[kLcRows];
#pragma unroll
    for (int k = 0; k < kLcRows; ++k) q[k] = p.enc + (b0 + min(r0 + k, static_cast<uint64_t>(n) - 1)) * p.W;
    uint32_t a[kLcRows] = {};
#pragma unroll 4
    for (uint32_t w = 0; w < p.W; ++w) {
      const uint32_t cw = cok ? p.cvt[static_cast<uint64_t>(w) * p.C + c] : 0u;
#pragma unroll
      for (int k = 0; k < kLcRows; ++k) a[k] += __popc(__ldg(q[k] + w) ^ cw);
    }
#pragma unroll
    for (int k = 0; k < kLcRows; ++k) {
      const uint64_t r = r0 + k;
      if (r >= n) break;
      unsigned long long key = cok ? (static_cast<unsigned long long>(a[k]) << 32) | c : ~0ull;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long other = __shfl_xor_sync(kFull, key, o);
        key = other < key ? other : key;
      }
      if (lane == 0) atomicMin(p.best + r, key);
      if (cok && static_cast<int32_t>(c) == p.labels[b0 + r]) p.truep[r] = a[k];
    }
  }
}

// ------------------------------------------------------------- binarise ----
__device__ __forceinline__ void binarize_store(const OnlineParams& p, uint32_t c, uint32_t j, bool col, double a,
                                               double total, uint32_t lane) {
  if (col) p.acc[static_cast<uint64_t>(c) * p.D + j] = a;
  const uint32_t wi = min(j >> 5, p.W - 1);
  uint32_t bit = 0;
  if (col) {
    const double twice = 2.0 * a;
    bit = twice > total ? 1u : (twice < total ? 0u : ((p.tie[wi] >> lane) & 1u));
  }
  const uint32_t word = __ballot_sync(kFull, bit);
  if (lane == 0 && (j >> 5) < p.W) {
    p.cv[static_cast<uint64_t>(c) * p.W + (j >> 5)] = word;
    if (p.cvt) p.cvt[static_cast<uint64_t>(j >> 5) * p.C + c] = word;
  }
}

struct Smem {
  uint32_t words[2][kOChunk][kOWords];
  double val[2][kOChunk];
  uint8_t flag[2][kOChunk];  // MERGED: bit0 listed, bit1 true sample
  uint32_t warpcnt[kOReplay / 32];
  double weight;
};

// ------------------------------------------------------- MERGED replay ----
__device__ void replay_merged(const OnlineParams& p, Smem& s, uint64_t b0, uint32_t n, uint32_t par) {
  const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
  const uint32_t nwb = (p.W + kOWords - 1) / kOWords;
  const uint64_t items = static_cast<uint64_t>(p.C) * nwb;
  for (uint64_t item = blockIdx.x; item < items; item += gridDim.x) {
    const uint32_t c = static_cast<uint32_t>(item / nwb);
    const uint32_t wb = static_cast<uint32_t>(item % nwb);
    const uint32_t j = wb * kOReplay + tid;
    const bool col = tid < kOReplay && j < p.D;
    double a = col ? p.acc[static_cast<uint64_t>(c) * p.D + j] : 0.0;
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
      if (tid < kOChunk && r < n) {
        const int32_t y = p.labels[b0 + r];
        const unsigned long long bst = p.best[r];
        const bool is_t = y == static_cast<int32_t>(c);
        const bool is_p = !is_t && static_cast<uint32_t>(bst) == c;
        if (is_t) rv = delta_of(p.truep[r], p.D);
        if (is_p) rv = penalty_of(bst, p.gamma, p.D);
        rf = (is_t || is_p ? 1 : 0) | (is_t ? 2 : 0);
      }
#pragma unroll
      for (int i = 0; i < kLoadsPer; ++i) {
        const uint32_t e = tid + i * kOThreads;
        const uint32_t k = e / kOWords, ww = e % kOWords;
        const uint32_t w = wb * kOWords + ww;
        rw[i] = (k < kOChunk && ch + k < n && w < p.W) ? __ldg(p.enc + (b0 + ch + k) * p.W + w) : 0u;
      }
    };
    auto store_chunk = [&](uint32_t buf) {
      if (tid < kOChunk) {
        s.val[buf][tid] = rv;
        s.flag[buf][tid] = rf;
      }
      mine |= rf & 1u;
#pragma unroll
      for (int i = 0; i < kLoadsPer; ++i) {
        const uint32_t e = tid + i * kOThreads;
        const uint32_t k = e / kOWords, ww = e % kOWords;
        if (k < kOChunk) s.words[buf][k][ww] = rw[i];
      }
    };
    load_chunk(0);
    store_chunk(0);
    __syncthreads();
    uint32_t buf = 0;
    for (uint32_t ch = 0; ch < n; ch += kOChunk, buf ^= 1u) {
      const bool more = ch + kOChunk < n;
      if (more) load_chunk(ch + kOChunk);  // in flight during the replay below
      const uint32_t m = min(static_cast<uint32_t>(kOChunk), n - ch);
      // branch-free replay: non-listed rows carry value +0.0, and adding +0.0
      // leaves every accumulator bit-identical (acc is never -0.0: it starts
      // from counts and x + y == 0 rounds to +0.0)
      if (tid < kOReplay) {
        const uint32_t ww = warp, sh = lane;
#pragma unroll 8
        for (uint32_t k = 0; k < m; ++k) {
          const uint32_t wd = s.words[buf][k][ww];
          const double v = s.val[buf][k];
          a = __dadd_rn(a, ((wd >> sh) & 1u) ? v : 0.0);
        }
      } else if (lane == 0) {
#pragma unroll 8
        for (uint32_t k = 0; k < m; ++k) {
          const uint8_t f = s.flag[buf][k];
          wsum = __dadd_rn(wsum, (f & 2u) ? s.val[buf][k] : 0.0);
          ntrue += f >> 1;
        }
      }
      if (more) store_chunk(buf ^ 1u);  // the other buffer was last read before the previous barrier
      __syncthreads();
    }
    if (tid == kOReplay) s.weight = wsum;
    const int touched = __syncthreads_or(mine);
    if (touched && tid < kOReplay) binarize_store(p, c, j, col, a, s.weight, lane);
    if (wb == 0 && tid == kOReplay) {
      p.weight[(par ^ 1u) * p.C + c] = wsum;
      p.counts[c] += ntrue;
    }
    __syncthreads();  // s.weight reuse by the next item
  }
}

// -------------------------------------------------------- LISTS phases ----
__device__ void build_lists(const OnlineParams& p, Smem& s, uint64_t b0, uint32_t n) {
  const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
  for (uint32_t c = blockIdx.x; c < p.C; c += gridDim.x) {
    double wsum = p.weight[c];
    uint64_t ntrue = 0;
    uint32_t len = 0;
    for (uint32_t ch = 0; ch < n; ch += kOChunk) {
      bool is_t = false, is_p = false;
      double v = 0.0;
      const uint32_t r = ch + tid;
      if (tid < kOChunk && r < n) {
        const int32_t y = p.labels[b0 + r];
        const unsigned long long bst = p.best[r];
        is_t = y == static_cast<int32_t>(c);
        is_p = !is_t && static_cast<uint32_t>(bst) == c;
        if (is_t) v = delta_of(p.truep[r], p.D);
        if (is_p) v = penalty_of(bst, p.gamma, p.D);
      }
      const bool flag = is_t || is_p;
      const uint32_t bal = __ballot_sync(kFull, flag);
      if (warp < kOChunk / 32 && lane == 0) s.warpcnt[warp] = __popc(bal);
      __syncthreads();
      uint32_t m = 0, off = 0;
#pragma unroll
      for (int k = 0; k < kOChunk / 32; ++k) {
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
      if (tid == kOReplay) {  // class weight over the true samples, in sample order
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
      p.weight[c] = wsum;
      p.counts[c] += ntrue;
      p.llen[c] = len;
    }
  }
}

__device__ void replay_lists(const OnlineParams& p, Smem& s, uint64_t b0) {
  const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
  const uint32_t nwb = (p.W + kOWords - 1) / kOWords;
  const uint64_t items = static_cast<uint64_t>(p.C) * nwb;
  for (uint64_t item = blockIdx.x; item < items; item += gridDim.x) {
    const uint32_t c = static_cast<uint32_t>(item / nwb);
    const uint32_t len = p.llen[c];
    if (len == 0) continue;  // untouched class: acc and class vector unchanged
    const uint32_t wb = static_cast<uint32_t>(item % nwb);
    const uint32_t j = wb * kOReplay + tid;
    const bool col = tid < kOReplay && j < p.D;
    double a = col ? p.acc[static_cast<uint64_t>(c) * p.D + j] : 0.0;
    const uint32_t* li = p.lidx + static_cast<uint64_t>(c) * p.bsz;
    const double* lv = p.lval + static_cast<uint64_t>(c) * p.bsz;
    uint32_t rw[kLoadsPer];
    double rv = 0.0;
    auto load_chunk = [&](uint32_t k0) {
      const uint32_t m = min(static_cast<uint32_t>(kOChunk), len - k0);
      if (tid < m) rv = lv[k0 + tid];
#pragma unroll
      for (int i = 0; i < kLoadsPer; ++i) {
        const uint32_t e = tid + i * kOThreads;
        const uint32_t k = e / kOWords, ww = e % kOWords;
        const uint32_t w = wb * kOWords + ww;
        rw[i] = (k < m && w < p.W) ? __ldg(p.enc + (b0 + li[k0 + k]) * p.W + w) : 0u;
      }
    };
    auto store_chunk = [&](uint32_t buf) {
      if (tid < kOChunk) s.val[buf][tid] = rv;
#pragma unroll
      for (int i = 0; i < kLoadsPer; ++i) {
        const uint32_t e = tid + i * kOThreads;
        const uint32_t k = e / kOWords, ww = e % kOWords;
        if (k < kOChunk) s.words[buf][k][ww] = rw[i];
      }
    };
    load_chunk(0);
    store_chunk(0);
    __syncthreads();
    uint32_t buf = 0;
    for (uint32_t k0 = 0; k0 < len; k0 += kOChunk, buf ^= 1u) {
      const bool more = k0 + kOChunk < len;
      if (more) load_chunk(k0 + kOChunk);
      const uint32_t m = min(static_cast<uint32_t>(kOChunk), len - k0);
      if (tid < kOReplay) {
        const uint32_t ww = warp, sh = lane;
#pragma unroll 8
        for (uint32_t k = 0; k < m; ++k) {
          const uint32_t wd = s.words[buf][k][ww];
          const double v = s.val[buf][k];
          a = __dadd_rn(a, ((wd >> sh) & 1u) ? v : 0.0);
        }
      }
      if (more) store_chunk(buf ^ 1u);
      __syncthreads();
    }
    if (tid < kOReplay) binarize_store(p, c, j, col, a, p.weight[c], lane);
  }
}

template <bool MERGED>
__global__ void __launch_bounds__(kOThreads) online_persistent_kernel(OnlineParams p) {
  cg::grid_group grid = cg::this_grid();
  __shared__ Smem s;
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  const uint64_t gwarps = static_cast<uint64_t>(gridDim.x) * (kOThreads / 32);
  const uint64_t gwarp = static_cast<uint64_t>(blockIdx.x) * (kOThreads / 32) + warp;
  const bool lane_class = p.C >= kLaneClassMinC;
  uint32_t par = 0;
  for (uint64_t b0 = 0; b0 < p.rows; b0 += p.bsz, par ^= 1u) {
    const uint32_t n = static_cast<uint32_t>(min(p.bsz, p.rows - b0));
    if (lane_class) {
      score_lane_class(p, b0, n, gwarp, gwarps, lane);
    } else {
      score_warp_per_row(p, b0, n, gwarp, gwarps, lane);
    }
    grid.sync();
    if constexpr (MERGED) {
      replay_merged(p, s, b0, n, par);
    } else {
      build_lists(p, s, b0, n);
      grid.sync();
      replay_lists(p, s, b0);
    }
    if (lane_class) {  // the atomicMin targets of the next batch
      const uint64_t gt = static_cast<uint64_t>(blockIdx.x) * kOThreads + threadIdx.x;
      for (uint64_t r = gt; r < p.bsz; r += static_cast<uint64_t>(gridDim.x) * kOThreads) p.best[r] = ~0ull;
    }
    grid.sync();
  }
}

__global__ void transpose_cv_kernel(const uint32_t* __restrict__ cv, uint32_t C, uint32_t W, uint32_t* __restrict__ cvt) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < static_cast<uint64_t>(C) * W;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t c = i / W, w = i % W;
    cvt[w * C + c] = cv[i];
  }
}

__global__ void weight_copy_kernel(const double* __restrict__ src, double* __restrict__ dst, uint32_t C) {
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < C) dst[c] = src[c];
}

template <bool MERGED>
unsigned cooperative_grid(hv_context* ctx, uint64_t want) {
  int per_sm = 0;
  ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, online_persistent_kernel<MERGED>, kOThreads, 0),
     "occupancy");
  if (per_sm < 1) fail(HV_ERR_CUDA, "online_persistent_kernel does not fit on an SM");
  return static_cast<unsigned>(std::max<uint64_t>(
      1, std::min<uint64_t>(want, static_cast<uint64_t>(ctx->sm_count) * static_cast<uint64_t>(per_sm))));
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
  const bool merged = C <= kMergedMaxC;
  const bool lane_class = C >= kLaneClassMinC;
  DevBuf<double> wts(2 * C, st), lval(merged ? 0 : C * n, st);
  DevBuf<unsigned long long> best(n, st);
  DevBuf<uint32_t> truep(n, st), lidx(merged ? 0 : C * n, st), llen(merged ? 0 : C, st), cvt(lane_class ? C * W : 0, st);
  weight_copy_kernel<<<grid_for(C, 128), 128, 0, st>>>(weight, wts.ptr, static_cast<uint32_t>(C));
  launched("weight_copy_kernel");
  if (lane_class) {
    ck(cudaMemsetAsync(best.ptr, 0xFF, n * sizeof(unsigned long long), st), "memset");
    transpose_cv_kernel<<<grid_for(C * W, 256, ctx->sm_count * 8), 256, 0, st>>>(cv, static_cast<uint32_t>(C),
                                                                                static_cast<uint32_t>(W), cvt.ptr);
    launched("transpose_cv_kernel");
  }
  const uint64_t items = static_cast<uint64_t>(C) * ((W + kOWords - 1) / kOWords);
  const uint64_t score_ctas = (n + kOThreads / 32 - 1) / (kOThreads / 32);
  const uint64_t want = std::max<uint64_t>(items, score_ctas);
  OnlineParams p{enc,     labels,   rows,     static_cast<uint32_t>(D), static_cast<uint32_t>(W),
                 static_cast<uint32_t>(C), n, gamma, tie, acc, wts.ptr, counts, cv, lane_class ? cvt.ptr : nullptr,
                 best.ptr, truep.ptr, lidx.ptr, lval.ptr, llen.ptr};
  void* args[] = {&p};
  if (merged) {
    const unsigned grid = cooperative_grid<true>(ctx, want);
    ck(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(online_persistent_kernel<true>), dim3(grid),
                                   dim3(kOThreads), args, 0, st),
       "online_persistent_kernel");
  } else {
    const unsigned grid = cooperative_grid<false>(ctx, want);
    ck(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(online_persistent_kernel<false>), dim3(grid),
                                   dim3(kOThreads), args, 0, st),
       "online_persistent_kernel");
  }
  launched("online_persistent_kernel");
  // MERGED leaves the final weights in the parity row after the last batch
  const size_t nb = (rows + n - 1) / n;
  const double* fin = merged ? wts.ptr + (nb & 1) * C : wts.ptr;
  weight_copy_kernel<<<grid_for(C, 128), 128, 0, st>>>(fin, weight, static_cast<uint32_t>(C));
  launched("weight_copy_kernel");
}

}  // namespace hvb
