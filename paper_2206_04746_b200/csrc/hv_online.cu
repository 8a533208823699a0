// hv_online.cu — the online trainer (model.cpp:250-301, Hamming metric) as
// ONE persistent cooperative kernel over all batches.
//
// The trainer is a chain of dependent batches: batch b is scored against the
// class vectors left by batch b-1, and every fp64 accumulator element must see
// the reference's sample-ordered in-place additions (model.cpp:54-63) to stay
// bit-identical. Per batch the work is small (at CHB-MIT: 1,024 rows, two
// classes) and latency-bound, so three kernel launches per batch plus
// L2-latency-bound replays dominated (profiles/configs_r1.jsonl: 180 us per
// batch). Here one launch runs every batch:
//
//   phase 1  score    warp per row: Hamming popcounts against every class
//                     vector, argmin (strict <, lowest class), delta_true and
//                     the wrong-class penalty -gamma (1 - delta_pred)
//   grid.sync
//   phase 2  update   item = (class c, 8-word block): streams the batch in
//                     256-row chunks; the chunk's entries of class c are
//                     compacted in row order into shared memory together with
//                     the 8 words of each listed row (all loads in flight at
//                     once), then thread j replays them on its register-held
//                     acc[c][j] while a ninth warp advances the class weight
//                     in the same order; touched classes are re-binarised with
//                     the batch's final weight (model.cpp:139-163, 277-279)
//   grid.sync
//
// Class weights are double-buffered per batch parity: every item of class c
// reads the batch-start weight and replays the same chain; the item with word
// block 0 publishes the result for the next batch.
#include <cooperative_groups.h>

#include <algorithm>

#include "hv_internal.cuh"

namespace cg = cooperative_groups;

namespace hvb {
namespace {

constexpr uint32_t kFull = 0xFFFFFFFFu;
constexpr int kOWords = 8;                       // words per update item
constexpr int kOChunk = 256;                     // batch rows per list chunk
constexpr int kOReplay = kOWords * 32;           // replay threads (one per bit column)
constexpr int kOThreads = kOReplay + 32;         // + one warp for the weight chain

struct OnlineParams {
  const uint32_t* enc;
  const int32_t* labels;
  uint64_t rows;
  uint32_t D, W, C;
  uint64_t bsz;
  double gamma;
  const uint32_t* tie;
  double* acc;       // C x D
  double* wpp;       // 2 x C class weights (batch-parity ping-pong)
  uint64_t* counts;  // C
  uint32_t* cv;      // C x W
  int32_t* pred;     // bsz scratch
  double* dt;        // bsz scratch: delta of the true class
  double* pen;       // bsz scratch: penalty for the predicted class
};

__global__ void __launch_bounds__(kOThreads) online_persistent_kernel(OnlineParams p) {
  cg::grid_group grid = cg::this_grid();
  __shared__ uint32_t s_words[kOChunk][kOWords];
  __shared__ double s_val[kOChunk];
  __shared__ uint32_t s_idx[kOChunk];
  __shared__ uint8_t s_true[kOChunk];
  __shared__ uint32_t s_warp[kOReplay / 32];
  __shared__ double s_weight;
  const uint32_t tid = threadIdx.x;
  const uint32_t lane = tid & 31u, warp = tid >> 5;
  const uint32_t nwb = (p.W + kOWords - 1) / kOWords;
  const uint64_t items = static_cast<uint64_t>(p.C) * nwb;
  const uint64_t gwarps = static_cast<uint64_t>(gridDim.x) * (kOThreads / 32);
  const uint64_t gwarp = static_cast<uint64_t>(blockIdx.x) * (kOThreads / 32) + warp;
  uint32_t par = 0;
  for (uint64_t b0 = 0; b0 < p.rows; b0 += p.bsz, par ^= 1u) {
    const uint32_t n = static_cast<uint32_t>(min(p.bsz, p.rows - b0));
    // ---- phase 1: score every row of the batch against the snapshot ----
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
        p.pred[r] = static_cast<int32_t>(best);
        p.dt[r] = static_cast<double>(truep) / static_cast<double>(p.D);
        const double dw = static_cast<double>(bestp) / static_cast<double>(p.D);
        p.pen[r] = __dmul_rn(-p.gamma, __dsub_rn(1.0, dw));
      }
    }
    grid.sync();
    // ---- phase 2: ordered per-class replay on (class, word block) items ----
    for (uint64_t item = blockIdx.x; item < items; item += gridDim.x) {
      const uint32_t c = static_cast<uint32_t>(item / nwb);
      const uint32_t wb = static_cast<uint32_t>(item % nwb);
      const uint32_t j = wb * kOReplay + tid;  // bit column of replay threads
      const bool col = tid < kOReplay && j < p.D;
      double a = col ? p.acc[static_cast<uint64_t>(c) * p.D + j] : 0.0;
      double wsum = p.wpp[par * p.C + c];
      uint64_t ntrue = 0;
      uint32_t touched = 0;
      for (uint32_t ch = 0; ch < n; ch += kOChunk) {
        // compact this chunk's entries of class c, in row order
        bool is_t = false, is_p = false;
        double v = 0.0;
        const uint32_t r = ch + tid;
        if (tid < kOChunk && r < n) {
          const int32_t y = p.labels[b0 + r];
          is_t = y == static_cast<int32_t>(c);
          is_p = !is_t && p.pred[r] == static_cast<int32_t>(c);
          if (is_t) v = p.dt[r];
          if (is_p) v = p.pen[r];
        }
        const bool flag = is_t || is_p;
        const uint32_t bal = __ballot_sync(kFull, flag);
        if (warp < kOChunk / 32 && lane == 0) s_warp[warp] = __popc(bal);
        __syncthreads();
        uint32_t m = 0, off = 0;
#pragma unroll
        for (int k = 0; k < kOChunk / 32; ++k) {
          off += (static_cast<uint32_t>(k) < warp) ? s_warp[k] : 0u;
          m += s_warp[k];
        }
        if (flag) {
          const uint32_t pos = off + __popc(bal & ((1u << lane) - 1u));
          s_idx[pos] = r;
          s_val[pos] = v;
          s_true[pos] = is_t ? 1 : 0;
        }
        __syncthreads();
        if (m == 0) continue;  // uniform: every thread read the same counts
        touched = 1;
        // the listed rows' words of this block, all loads in flight together
        for (uint32_t e = tid; e < m * kOWords; e += kOThreads) {
          const uint32_t k = e / kOWords, ww = e % kOWords;
          const uint32_t w = wb * kOWords + ww;
          s_words[k][ww] = w < p.W ? __ldg(p.enc + (b0 + s_idx[k]) * p.W + w) : 0u;
        }
        __syncthreads();
        if (tid < kOReplay) {
          const uint32_t ww = warp, sh = lane;
          for (uint32_t k = 0; k < m; ++k) {
            if ((s_words[k][ww] >> sh) & 1u) a = __dadd_rn(a, s_val[k]);
          }
        } else if (lane == 0) {
          for (uint32_t k = 0; k < m; ++k) {
            if (s_true[k]) {
              wsum = __dadd_rn(wsum, s_val[k]);
              ++ntrue;
            }
          }
        }
        __syncthreads();  // smem is rewritten by the next chunk
      }
      if (tid == kOReplay) s_weight = wsum;
      __syncthreads();
      if (touched) {
        if (col) p.acc[static_cast<uint64_t>(c) * p.D + j] = a;
        if (tid < kOReplay) {
          const double total = s_weight;
          const uint32_t wi = min(j >> 5, p.W - 1);
          uint32_t bit = 0;
          if (col) {
            const double twice = 2.0 * a;
            bit = twice > total ? 1u : (twice < total ? 0u : ((p.tie[wi] >> lane) & 1u));
          }
          const uint32_t word = __ballot_sync(kFull, bit);
          if (lane == 0 && (j >> 5) < p.W) p.cv[static_cast<uint64_t>(c) * p.W + (j >> 5)] = word;
        }
      }
      if (wb == 0 && tid == kOReplay) {
        p.wpp[(par ^ 1u) * p.C + c] = s_weight;
        p.counts[c] += ntrue;
      }
      __syncthreads();  // s_weight / smem reuse by the next item
    }
    grid.sync();
  }
}

__global__ void copy_weight_kernel(const double* __restrict__ src, double* __restrict__ dst, uint32_t C) {
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < C) dst[c] = src[c];
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
  DevBuf<double> wpp(2 * C, st), dt(n, st), pen(n, st);
  DevBuf<int32_t> pred(n, st);
  copy_weight_kernel<<<grid_for(C, 128), 128, 0, st>>>(weight, wpp.ptr, static_cast<uint32_t>(C));
  launched("copy_weight_kernel");
  int per_sm = 0;
  ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, online_persistent_kernel, kOThreads, 0), "occupancy");
  if (per_sm < 1) fail(HV_ERR_CUDA, "online_persistent_kernel does not fit on an SM");
  const uint64_t items = static_cast<uint64_t>(C) * ((W + kOWords - 1) / kOWords);
  const uint64_t score_ctas = (n + kOThreads / 32 - 1) / (kOThreads / 32);
  const uint64_t want = std::max<uint64_t>(items, score_ctas);
  const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(want, static_cast<uint64_t>(ctx->sm_count) * per_sm));
  OnlineParams p{enc, labels, rows, static_cast<uint32_t>(D), static_cast<uint32_t>(W), static_cast<uint32_t>(C),
                 bsz, gamma, tie, acc, wpp.ptr, counts, cv, pred.ptr, dt.ptr, pen.ptr};
  void* args[] = {&p};
  ck(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(online_persistent_kernel), dim3(grid), dim3(kOThreads), args,
                                 0, st),
     "online_persistent_kernel");
  launched("online_persistent_kernel");
  // final weight: parity after the last batch
  const size_t nb = (rows + bsz - 1) / bsz;
  copy_weight_kernel<<<grid_for(C, 128), 128, 0, st>>>(wpp.ptr + (nb & 1) * C, weight, static_cast<uint32_t>(C));
  launched("copy_weight_kernel");
}

}  // namespace hvb
