// hv_model.cu — classical trainer, online trainer and nearest-class scan
// (reference model.cpp:24-320).
//
// Classical training (model.cpp:219-244) is a per-class vertical bit count:
// rows are bucketed by label with a warp-aggregated counting sort, then the
// shared column-count kernel streams each class's rows once (Harley–Seal
// counters, HBM bound). Counts are exact uint32; accumulators are their
// double values, exactly like the reference.
//
// Online training (model.cpp:250-301) must reproduce fp64 rounding exactly.
// The reference adds each sample's weight into acc[class][j] in place, in
// sample order. Here every (class, position) element is owned by one thread
// that walks the class's ordered update list for the batch, so each element
// sees the same sequence of IEEE additions (__dadd_rn, no contraction) and
// the result is bit-identical. Scores of a batch are computed against the
// batch-start class vectors (the snapshot, model.cpp:246-248) before any
// update of that batch is applied.

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <limits>
#include <memory>
#include <vector>

#include "hv_internal.cuh"
#include "hv_scan.cuh"
#include "hv_scan_mma.cuh"
#include "hv_scan_tc.cuh"
#include "hv_stage.h"

namespace hvb {

constexpr uint32_t FULL = 0xFFFFFFFFu;

// ------------------------------------------------- label bucketing ----
// model.cpp:24-37 check_labels (range), plus per-class histogram.
__global__ void label_hist_kernel(const int32_t* __restrict__ y, uint64_t n, uint32_t C, uint32_t* __restrict__ hist,
                                  unsigned long long* err) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t base = blockIdx.x * (uint64_t)blockDim.x + (threadIdx.x & ~31u); base < n; base += stride) {
    const uint64_t i = base + lane;
    const bool valid = i < n;
    const int32_t lab = valid ? y[i] : -1;
    const bool ok = valid && lab >= 0 && static_cast<uint32_t>(lab) < C;
    if (valid && !ok) latch(err, kErrLabel, i);
    const uint32_t mask = __match_any_sync(FULL, ok ? lab : -1);
    if (ok && lane == static_cast<uint32_t>(__ffs(mask) - 1)) atomicAdd(hist + lab, __popc(mask));
  }
}

__global__ void label_scan_kernel(const uint32_t* __restrict__ hist, uint32_t C, uint64_t* __restrict__ offsets,
                                  uint64_t* __restrict__ class_rows, uint32_t* __restrict__ cursor) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  uint64_t acc = 0;
  for (uint32_t c = 0; c < C; ++c) {
    offsets[c] = acc;
    acc += hist[c];
    if (class_rows) class_rows[c] += hist[c];
    cursor[c] = 0;
  }
  offsets[C] = acc;
}

__global__ void label_scatter_kernel(const int32_t* __restrict__ y, uint64_t n, uint32_t C,
                                     const uint64_t* __restrict__ offsets, uint32_t* __restrict__ cursor,
                                     uint32_t* __restrict__ perm) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t base = blockIdx.x * (uint64_t)blockDim.x + (threadIdx.x & ~31u); base < n; base += stride) {
    const uint64_t i = base + lane;
    const bool valid = i < n;
    const int32_t lab = valid ? y[i] : -1;
    const bool ok = valid && lab >= 0 && static_cast<uint32_t>(lab) < C;
    const uint32_t mask = __match_any_sync(FULL, ok ? lab : -1);
    const uint32_t leader = __ffs(mask) - 1;
    uint32_t start = 0;
    if (ok && lane == leader) start = atomicAdd(cursor + lab, __popc(mask));
    start = __shfl_sync(FULL, start, leader);
    if (ok) {
      const uint32_t rank = __popc(mask & ((1u << lane) - 1u));
      perm[offsets[lab] + start + rank] = static_cast<uint32_t>(i);
    }
  }
}

// bit = 2c > n ? 1 : 2c < n ? 0 : tie   (model.cpp:139-163 with acc = count, weight = n)
__global__ void binarize_counts_kernel(const uint32_t* __restrict__ counts, const uint64_t* __restrict__ class_rows,
                                       uint32_t C, uint32_t D, uint32_t W, const uint32_t* __restrict__ tie,
                                       uint32_t* __restrict__ cv) {
  const uint64_t total = static_cast<uint64_t>(C) * W;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t c = static_cast<uint32_t>(i / W);
    const uint32_t w = static_cast<uint32_t>(i % W);
    const uint64_t n = class_rows[c];
    const uint32_t* cc = counts + static_cast<uint64_t>(c) * 32u * W + 32u * w;
    const uint32_t tw = tie[w];
    uint32_t word = 0;
#pragma unroll 8
    for (int t = 0; t < 32; ++t) {
      const uint64_t twice = 2ull * cc[t];
      const uint32_t bit = twice > n ? 1u : (twice < n ? 0u : ((tw >> t) & 1u));
      word |= bit << t;
    }
    cv[i] = word & valid_mask(w, D);
  }
}

// acc[c][j] = double(count), weight = count = rows of class c
__global__ void init_from_counts_kernel(const uint32_t* __restrict__ counts, const uint64_t* __restrict__ class_rows,
                                        uint32_t C, uint32_t D, uint32_t W, double* __restrict__ acc,
                                        double* __restrict__ weight, uint64_t* __restrict__ cnt) {
  const uint64_t total = static_cast<uint64_t>(C) * D;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t c = i / D;
    const uint64_t j = i % D;
    acc[i] = static_cast<double>(counts[c * 32ull * W + j]);
    if (j == 0) {
      weight[c] = static_cast<double>(class_rows[c]);
      cnt[c] = class_rows[c];
    }
  }
}

// model.cpp:139-163 for the classes with touched[c] != 0 (or all when touched == nullptr)
__global__ void refresh_kernel(const double* __restrict__ acc, const double* __restrict__ weight,
                               const uint32_t* __restrict__ touched, uint32_t C, uint32_t D, uint32_t W,
                               const uint32_t* __restrict__ tie, uint32_t* __restrict__ cv) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint64_t warps_total = static_cast<uint64_t>(C) * W;
  const uint64_t stride = (uint64_t)gridDim.x * (blockDim.x >> 5);
  for (uint64_t t = blockIdx.x * (uint64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); t < warps_total; t += stride) {
    const uint32_t c = static_cast<uint32_t>(t / W);
    const uint32_t w = static_cast<uint32_t>(t % W);
    if (touched && touched[c] == 0) continue;
    const uint32_t j = w * 32u + lane;
    uint32_t bit = 0;
    if (j < D) {
      const double twice = 2.0 * acc[static_cast<uint64_t>(c) * D + j];
      const double total = weight[c];
      bit = twice > total ? 1u : (twice < total ? 0u : ((tie[w] >> lane) & 1u));
    }
    const uint32_t word = __ballot_sync(FULL, bit);
    if (lane == 0) cv[t] = word;
  }
}

// ------------------------------------------------------ Hamming scan ----
// model.cpp:303-320 + 69-79 + 96-104: one warp per query row, C popcounts of
// row ^ class_vector reduced with REDUX; argmin with strict < (lowest class
// wins ties). Integer popcounts order exactly like popc/D doubles.
//
// HBM-bound at few classes (CHB-MIT: 2 x 313 POPC per 1,256-byte row), so the
// row is streamed with U independent word loads in flight per lane
// (evict-first: rows are read once); CB classes are scored per pass over the
// row, class words come from L1.
template <int CB, int U>
__global__ void __launch_bounds__(256) predict_hamming_kernel(const uint32_t* __restrict__ cv, uint32_t C, uint32_t D,
                                                              uint32_t W, uint32_t ldq,
                                                              const uint32_t* __restrict__ enc, uint64_t rows,
                                                              int32_t* __restrict__ labels, double* __restrict__ dist,
                                                              uint32_t* __restrict__ pops) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint64_t stride = (uint64_t)gridDim.x * (blockDim.x >> 5);
  for (uint64_t r = blockIdx.x * (uint64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); r < rows; r += stride) {
    const uint32_t* q = enc + r * ldq;
    uint32_t best = 0, bestp = 0xFFFFFFFFu;
    for (uint32_t c0 = 0; c0 < C; c0 += CB) {
      uint32_t acc[CB];
#pragma unroll
      for (int k = 0; k < CB; ++k) acc[k] = 0;
      for (uint32_t w0 = 0; w0 < W; w0 += 32u * U) {
        uint32_t x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t w = w0 + lane + 32u * u;
          x[u] = w < W ? __ldcs(q + w) : 0u;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t w = w0 + lane + 32u * u;
          if (w < W) {
#pragma unroll
            for (int k = 0; k < CB; ++k) {
              if (c0 + k < C) acc[k] += __popc(x[u] ^ __ldg(cv + static_cast<uint64_t>(c0 + k) * W + w));
            }
          }
        }
      }
#pragma unroll
      for (int k = 0; k < CB; ++k) {
        const uint32_t tot = __reduce_add_sync(FULL, acc[k]);
        const uint32_t c = c0 + k;
        if (c < C) {
          if (tot < bestp) {
            bestp = tot;
            best = c;
          }
          if (lane == (c & 31u)) {
            if (pops) pops[r * C + c] = tot;
            if (dist) dist[r * C + c] = static_cast<double>(tot) / static_cast<double>(D);
          }
        }
      }
    }
    if (lane == 0 && labels) labels[r] = static_cast<int32_t>(best);
  }
}

// The same scan over pitched, 16-byte aligned query rows (the engine's own
// layout, ldq % 4 == 0): each lane reads whole uint4s of the row (U = 3 in
// flight: 96 words per lane-round), the class vectors are staged once per CTA
// in shared memory at pitch W4 = ceil(W / 4) uint4s with zero padding, and
// the words of the last uint4 past W are masked (the row padding is never
// written by the encoder). scripts/probe_stream.cu at CHB-MIT: 6.1-6.2 TB/s
// against 4.1 for 4-byte loads of unpitched rows.
template <int CB>
__global__ void __launch_bounds__(256) predict_hamming_pitched_kernel(
    const uint32_t* __restrict__ cv, uint32_t C, uint32_t D, uint32_t W, uint32_t ldq, const uint32_t* __restrict__ enc,
    uint64_t rows, int32_t* __restrict__ labels, double* __restrict__ dist, uint32_t* __restrict__ pops) {
  constexpr int U = 3;
  extern __shared__ uint4 cvs[];  // [C][W4]
  const uint32_t W4 = (W + 3) / 4;
  uint32_t* cvw = reinterpret_cast<uint32_t*>(cvs);
  for (uint32_t i = threadIdx.x; i < C * W4 * 4; i += blockDim.x) {
    const uint32_t c = i / (W4 * 4), w = i % (W4 * 4);
    cvw[i] = w < W ? __ldg(cv + static_cast<uint64_t>(c) * W + w) : 0u;
  }
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t tail = W & 3u;  // valid words of the last uint4 (0 = all four)
  const uint64_t stride = (uint64_t)gridDim.x * (blockDim.x >> 5);
  for (uint64_t r = blockIdx.x * (uint64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); r < rows; r += stride) {
    const uint4* q = reinterpret_cast<const uint4*>(enc + r * ldq);
    uint32_t best = 0, bestp = 0xFFFFFFFFu;
    for (uint32_t c0 = 0; c0 < C; c0 += CB) {
      uint32_t acc[CB];
#pragma unroll
      for (int k = 0; k < CB; ++k) acc[k] = 0;
      for (uint32_t v0 = 0; v0 < W4; v0 += 32u * U) {
        uint4 x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t v = v0 + lane + 32u * u;
          x[u] = v < W4 ? __ldcs(q + v) : make_uint4(0, 0, 0, 0);
          if (v == W4 - 1 && tail) {
            if (tail < 4) x[u].w = 0;
            if (tail < 3) x[u].z = 0;
            if (tail < 2) x[u].y = 0;
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t v = v0 + lane + 32u * u;
          if (v < W4) {
#pragma unroll
            for (int k = 0; k < CB; ++k) {
              if (c0 + k < C) {
                const uint4 c = cvs[(c0 + k) * W4 + v];
                acc[k] += __popc(x[u].x ^ c.x) + __popc(x[u].y ^ c.y) + __popc(x[u].z ^ c.z) + __popc(x[u].w ^ c.w);
              }
            }
          }
        }
      }
#pragma unroll
      for (int k = 0; k < CB; ++k) {
        const uint32_t tot = __reduce_add_sync(FULL, acc[k]);
        const uint32_t c = c0 + k;
        if (c < C) {
          if (tot < bestp) {
            bestp = tot;
            best = c;
          }
          if (lane == (c & 31u)) {
            if (pops) pops[r * C + c] = tot;
            if (dist) dist[r * C + c] = static_cast<double>(tot) / static_cast<double>(D);
          }
        }
      }
    }
    if (lane == 0 && labels) labels[r] = static_cast<int32_t>(best);
  }
}

// Two classes, labels only (the CHB-MIT workload): popc(q^c1) < popc(q^c0)
// <=> 2 popc(d & (q ^ c0)) > popc(d) with d = c0 ^ c1 — on bits where the
// classes agree both distances count the same, where they differ exactly one
// does. One LOP3 + one POPC per word instead of two XOR + two POPC, so the
// scan stays on HBM instead of the XU pipe. Ties (2A == |d|) keep class 0, the
// reference's strict < (model.cpp:96-104). Pitched 16-byte rows.
__global__ void __launch_bounds__(256) predict_two_class_kernel(const uint32_t* __restrict__ cv, uint32_t W,
                                                                uint32_t ldq, const uint32_t* __restrict__ enc,
                                                                uint64_t rows, int32_t* __restrict__ labels) {
  constexpr int U = 3;
  extern __shared__ uint4 cd[];  // [W4] c0, then [W4] d = c0 ^ c1 (zero padded)
  const uint32_t W4 = (W + 3) / 4;
  uint32_t* cw = reinterpret_cast<uint32_t*>(cd);
  uint32_t dpop = 0;
  for (uint32_t w = threadIdx.x; w < W4 * 4; w += blockDim.x) {
    const uint32_t a = w < W ? __ldg(cv + w) : 0u, b = w < W ? __ldg(cv + W + w) : 0u;
    cw[w] = a;
    cw[W4 * 4 + w] = a ^ b;
  }
  __syncthreads();
  for (uint32_t w = threadIdx.x & 31u; w < W4 * 4; w += 32u) dpop += __popc(cw[W4 * 4 + w]);
  dpop = __reduce_add_sync(FULL, dpop);  // |d| (every warp computes it)
  const uint32_t lane = threadIdx.x & 31u;
  const uint64_t stride = (uint64_t)gridDim.x * (blockDim.x >> 5);
  for (uint64_t r = blockIdx.x * (uint64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); r < rows; r += stride) {
    const uint4* q = reinterpret_cast<const uint4*>(enc + r * ldq);
    uint32_t a = 0;
    for (uint32_t v0 = 0; v0 < W4; v0 += 32u * U) {
      uint4 x[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t v = v0 + lane + 32u * u;
        x[u] = v < W4 ? __ldcs(q + v) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t v = v0 + lane + 32u * u;
        if (v < W4) {
          // the row's padding words meet d's zero padding: no mask needed
          const uint4 c = cd[v], d = cd[W4 + v];
          a += __popc((x[u].x ^ c.x) & d.x) + __popc((x[u].y ^ c.y) & d.y) + __popc((x[u].z ^ c.z) & d.z) +
               __popc((x[u].w ^ c.w) & d.w);
        }
      }
    }
    a = __reduce_add_sync(FULL, a);
    if (lane == 0) labels[r] = 2 * a > dpop ? 1 : 0;
  }
}

// Many classes (C >= 32): CTA-tiled scan (hv_scan.cuh), 32 rows x 32 classes
// per tile, tiles ordered class-block-minor so the CTAs sharing a row tile run
// together (the rows stay in L2). Per-row argmin merged across class blocks
// with a 64-bit atomicMin on (popc << 32 | class) = the reference's strict-<
// argmin.
__global__ void __launch_bounds__(256) predict_tiled_kernel(const uint32_t* __restrict__ cv, uint32_t C, uint32_t D,
                                                            uint32_t W, const uint32_t* __restrict__ enc,
                                                            uint64_t rows, unsigned long long* __restrict__ best,
                                                            double* __restrict__ dist, uint32_t* __restrict__ pops) {
  __shared__ ScanSmem s;
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  const uint32_t ncb = (C + kScanCls - 1) / kScanCls;
  const uint64_t ntiles = (rows + kScanRows - 1) / kScanRows;
  for (uint64_t it = blockIdx.x; it < ntiles * ncb; it += gridDim.x) {
    const uint32_t cb = static_cast<uint32_t>(it % ncb);
    const uint64_t row0 = (it / ncb) * kScanRows;
    const uint32_t nr = static_cast<uint32_t>(min(static_cast<uint64_t>(kScanRows), rows - row0));
    uint32_t a[kScanRowsPerWarp];
    scan_tile<256>(enc, row0, nr, W, cv, C, cb * kScanCls, s, a);
    const uint32_t c = cb * kScanCls + lane;
#pragma unroll
    for (int k = 0; k < kScanRowsPerWarp; ++k) {
      const uint32_t r = warp * kScanRowsPerWarp + k;
      if (r >= nr) break;
      const uint64_t row = row0 + r;
      if (c < C) {
        if (pops) pops[row * C + c] = a[k];
        if (dist) dist[row * C + c] = static_cast<double>(a[k]) / static_cast<double>(D);
      }
      const unsigned long long key = warp_min_u64(c < C ? scan_key(a[k], c) : ~0ull);
      if (lane == 0) atomicMin(best + row, key);
    }
  }
}

// Many classes on the int8 tensor cores (hv_scan_mma.cuh): exact integer
// Hamming distances |q| + |c| - 2<q,c>; per-row argmin merged across warps
// and class tiles with the same 64-bit atomicMin key as the POPC scan.
__global__ void class_popcount_kernel(const uint32_t* __restrict__ cv, uint32_t C, uint32_t W,
                                      uint32_t* __restrict__ cpop) {
  const uint32_t lane = threadIdx.x & 31u;
  for (uint32_t c = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); c < C; c += gridDim.x * (blockDim.x >> 5)) {
    uint32_t a = 0;
    for (uint32_t w = lane; w < W; w += 32u) a += __popc(cv[static_cast<uint64_t>(c) * W + w]);
    a = __reduce_add_sync(FULL, a);
    if (lane == 0) cpop[c] = a;
  }
}

__global__ void __launch_bounds__(kMmaThreads) predict_imma_kernel(const uint32_t* __restrict__ cv, uint32_t C,
                                                                   uint32_t D, uint32_t W,
                                                                   const uint32_t* __restrict__ enc, uint64_t rows,
                                                                   const uint32_t* __restrict__ cpop,
                                                                   unsigned long long* __restrict__ best,
                                                                   double* __restrict__ dist,
                                                                   uint32_t* __restrict__ pops) {
  extern __shared__ __align__(16) uint8_t mma_dsm[];
  MmaSmem& s = *reinterpret_cast<MmaSmem*>(mma_dsm);
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  const uint32_t g = lane >> 2, qd = lane & 3u, wm = warp >> 1, wn = warp & 1u;
  const uint32_t nct = (C + kMmaCls - 1) / kMmaCls;
  const uint64_t nrt = (rows + kMmaRows - 1) / kMmaRows;
  for (uint64_t it = blockIdx.x; it < nrt * nct; it += gridDim.x) {
    const uint32_t c0 = static_cast<uint32_t>(it % nct) * kMmaCls;
    const uint64_t row0 = (it / nct) * kMmaRows;
    int acc[2][8][4];
    mma_scan_tile(enc, row0, rows, W, cv, C, c0, s, acc);
#pragma unroll
    for (int m = 0; m < 2; ++m) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint32_t r = wm * 32 + m * 16 + g + 8 * h;
        const uint64_t row = row0 + r;
        const uint32_t rp = s.rowpop[r];
        unsigned long long key = ~0ull;
#pragma unroll
        for (int t = 0; t < 8; ++t) {
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const uint32_t c = c0 + wn * 64 + t * 8 + 2 * qd + j;
            if (c < C && row < rows) {
              const uint32_t ham = rp + cpop[c] - 2u * static_cast<uint32_t>(acc[m][t][2 * h + j]);
              const unsigned long long k = (static_cast<unsigned long long>(ham) << 32) | c;
              key = k < key ? k : key;
              if (pops) pops[row * C + c] = ham;
              if (dist) dist[row * C + c] = static_cast<double>(ham) / static_cast<double>(D);
            }
          }
        }
#pragma unroll
        for (int o = 1; o < 4; o <<= 1) {
          const unsigned long long other = __shfl_xor_sync(FULL, key, o);
          key = other < key ? other : key;
        }
        if (qd == 0 && row < rows) atomicMin(best + row, key);
      }
    }
    __syncthreads();  // s.rowpop is reset by the next tile
  }
}

__global__ void best_to_labels_kernel(const unsigned long long* __restrict__ best, uint64_t rows,
                                      int32_t* __restrict__ labels) {
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < rows; r += (uint64_t)gridDim.x * blockDim.x) {
    labels[r] = static_cast<int32_t>(static_cast<uint32_t>(best[r]));
  }
}

// ------------------------------------------------------- cosine scan ----
// model.cpp:80-93, 40-51: exact sequential fp64 like the reference —
// norm_sq = sum_j acc^2 in j order; dot = sum over set bits in increasing j.
__global__ void class_norms_kernel(const double* __restrict__ acc, uint32_t C, uint32_t D, double* __restrict__ norm) {
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  const double* a = acc + static_cast<uint64_t>(c) * D;
  double s = 0.0;
  for (uint32_t j = 0; j < D; ++j) s = __dadd_rn(s, __dmul_rn(a[j], a[j]));
  norm[c] = s;
}

// one thread per (row, class): score = dot / (sqrt(norm) * sqrt(ones)), -inf for empty class
__global__ void cosine_scores_kernel(const double* __restrict__ acc, const double* __restrict__ norm, uint32_t C,
                                     uint32_t D, uint32_t W, const uint32_t* __restrict__ enc, uint64_t rows,
                                     double* __restrict__ scores, unsigned long long* err, uint64_t err_base) {
  const uint64_t total = rows * C;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t r = i / C;
    const uint32_t c = static_cast<uint32_t>(i % C);
    const uint32_t* q = enc + r * W;
    uint32_t ones = 0;
    for (uint32_t w = 0; w < W; ++w) ones += __popc(q[w]);
    if (ones == 0) {
      latch(err, kErrZeroQuery, err_base + r);
      scores[i] = 0.0;
      continue;
    }
    const double ns = norm[c];
    if (ns == 0.0) {
      scores[i] = -__longlong_as_double(0x7FF0000000000000ll);
      continue;
    }
    const double* a = acc + static_cast<uint64_t>(c) * D;
    double dot = 0.0;
    for (uint32_t w = 0; w < W; ++w) {
      uint32_t bits = q[w];
      while (bits) {
        const uint32_t t = __ffs(bits) - 1;
        dot = __dadd_rn(dot, a[w * 32u + t]);
        bits &= bits - 1;
      }
    }
    scores[i] = __ddiv_rn(dot, __dmul_rn(__dsqrt_rn(ns), __dsqrt_rn(static_cast<double>(ones))));
  }
}

// argmax with strict > (model.cpp:96-104), one thread per row
__global__ void argmax_kernel(const double* __restrict__ scores, uint64_t rows, uint32_t C, int32_t* __restrict__ labels) {
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < rows; r += (uint64_t)gridDim.x * blockDim.x) {
    const double* s = scores + r * C;
    uint32_t best = 0;
    for (uint32_t c = 1; c < C; ++c) {
      if (s[c] > s[best]) best = c;
    }
    labels[r] = static_cast<int32_t>(best);
  }
}

// ------------------------------------------------------------ online ----
// Per-sample scoring of one batch against the snapshot (model.cpp:259-265):
// predicted label, delta_true and the wrong-class penalty -gamma*(1-delta_wrong).
__global__ void online_score_hamming_kernel(const uint32_t* __restrict__ cv, uint32_t C, uint32_t D, uint32_t W,
                                            const uint32_t* __restrict__ batch, uint64_t rows,
                                            const int32_t* __restrict__ labels, double gamma,
                                            int32_t* __restrict__ pred, double* __restrict__ dtrue,
                                            double* __restrict__ pen) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint64_t stride = (uint64_t)gridDim.x * (blockDim.x >> 5);
  for (uint64_t r = blockIdx.x * (uint64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); r < rows; r += stride) {
    const uint32_t* q = batch + r * W;
    const int32_t y = labels[r];
    uint32_t best = 0, bestp = 0xFFFFFFFFu, truep = 0;
    for (uint32_t c = 0; c < C; ++c) {
      uint32_t a = 0;
      for (uint32_t w = lane; w < W; w += 32u) a += __popc(q[w] ^ cv[static_cast<uint64_t>(c) * W + w]);
      a = __reduce_add_sync(FULL, a);
      if (a < bestp) {
        bestp = a;
        best = c;
      }
      if (static_cast<int32_t>(c) == y) truep = a;
    }
    if (lane == 0) {
      pred[r] = static_cast<int32_t>(best);
      dtrue[r] = static_cast<double>(truep) / static_cast<double>(D);
      const double dw = static_cast<double>(bestp) / static_cast<double>(D);
      pen[r] = __dmul_rn(-gamma, __dsub_rn(1.0, dw));
    }
  }
}

// D-sliced online training (SURVEY.md §8e exact mode): partial Hamming
// popcounts of each batch row against each class over this rank's word slice
// (warp per row), summed across ranks by the caller's all-reduce.
__global__ void online_partial_popc_kernel(const uint32_t* __restrict__ cv, uint32_t C, uint32_t Ws,
                                           const uint32_t* __restrict__ batch, uint64_t rows,
                                           uint32_t* __restrict__ popc, uint32_t* const* peers, uint32_t npeers) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint64_t stride = (uint64_t)gridDim.x * (blockDim.x >> 5);
  for (uint64_t r = blockIdx.x * (uint64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); r < rows; r += stride) {
    const uint32_t* q = batch + r * Ws;
    for (uint32_t c = 0; c < C; ++c) {
      uint32_t a = 0;
      for (uint32_t w = lane; w < Ws; w += 32u) a += __popc(q[w] ^ cv[static_cast<uint64_t>(c) * Ws + w]);
      a = __reduce_add_sync(FULL, a);
      if (lane == 0) {
        if (peers) {  // fused with the reduction: add into every rank's buffer over peer memory
          for (uint32_t q = 0; q < npeers; ++q) atomicAdd_system(peers[q] + r * C + c, a);
        } else {
          popc[r * C + c] = a;
        }
      }
    }
  }
}

// Scores from full-row popcounts (rows x C): the same argmin (strict <, lowest
// class on ties, model.cpp:96-104) and doubles as online_score_hamming_kernel.
__global__ void online_score_popc_kernel(const uint32_t* __restrict__ popc, uint32_t C, uint32_t D, uint64_t rows,
                                         const int32_t* __restrict__ labels, double gamma, int32_t* __restrict__ pred,
                                         double* __restrict__ dtrue, double* __restrict__ pen,
                                         unsigned long long* __restrict__ err) {
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < rows; r += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t* pc = popc + r * C;
    const int32_t y = labels[r];
    uint32_t best = 0, bestp = pc[0];
    for (uint32_t c = 1; c < C; ++c) {
      if (pc[c] < bestp) {
        bestp = pc[c];
        best = c;
      }
    }
    uint32_t truep = 0;
    if (y < 0 || static_cast<uint32_t>(y) >= C) {
      latch(err, kErrLabel, r);
    } else {
      truep = pc[y];
    }
    pred[r] = static_cast<int32_t>(best);
    dtrue[r] = static_cast<double>(truep) / static_cast<double>(D);
    const double dw = static_cast<double>(bestp) / static_cast<double>(D);
    pen[r] = __dmul_rn(-gamma, __dsub_rn(1.0, dw));
  }
}

// Cosine variant: scores already computed (rows x C); model.cpp:109-113 score_to_delta.
__global__ void online_score_cosine_kernel(const double* __restrict__ scores, uint32_t C, uint64_t rows,
                                           const int32_t* __restrict__ labels, double gamma,
                                           int32_t* __restrict__ pred, double* __restrict__ dtrue,
                                           double* __restrict__ pen) {
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < rows; r += (uint64_t)gridDim.x * blockDim.x) {
    const double* s = scores + r * C;
    uint32_t best = 0;
    for (uint32_t c = 1; c < C; ++c) {
      if (s[c] > s[best]) best = c;
    }
    auto to_delta = [](double v) { return isinf(v) ? 1.0 : __ddiv_rn(__dsub_rn(1.0, v), 2.0); };
    pred[r] = static_cast<int32_t>(best);
    dtrue[r] = to_delta(s[labels[r]]);
    pen[r] = __dmul_rn(-gamma, __dsub_rn(1.0, to_delta(s[best])));
  }
}

// One warp per class: the ordered list of (sample, value) updates hitting the
// class in this batch, and the class weight advanced in sample order
// (model.cpp:266-274). weight_out/counts_out are updated in place (delta
// mode passes zeroed arrays).
__global__ void online_lists_kernel(const int32_t* __restrict__ labels, const int32_t* __restrict__ pred,
                                    const double* __restrict__ dtrue, const double* __restrict__ pen, uint64_t rows,
                                    uint32_t C, uint32_t cap, uint32_t* __restrict__ idx, double* __restrict__ val,
                                    uint32_t* __restrict__ len, double* __restrict__ weight,
                                    uint64_t* __restrict__ counts, uint32_t* __restrict__ touched) {
  const uint32_t c = blockIdx.x;
  const uint32_t lane = threadIdx.x;
  if (c >= C) return;
  uint32_t n = 0, ntrue = 0;
  double wsum = weight[c];
  for (uint64_t i0 = 0; i0 < rows; i0 += 32) {
    const uint64_t i = i0 + lane;
    const bool valid = i < rows;
    const int32_t y = valid ? labels[i] : -1;
    const int32_t p = valid ? pred[i] : -1;
    const bool is_true = y == static_cast<int32_t>(c);
    const bool is_pen = !is_true && p == static_cast<int32_t>(c);
    const double dt = is_true ? dtrue[i] : 0.0;
    const uint32_t m = __ballot_sync(FULL, is_true || is_pen);
    if (is_true || is_pen) {
      const uint32_t pos = n + __popc(m & ((1u << lane) - 1u));
      idx[static_cast<uint64_t>(c) * cap + pos] = static_cast<uint32_t>(i);
      val[static_cast<uint64_t>(c) * cap + pos] = is_true ? dt : pen[i];
    }
    n += __popc(m);
    uint32_t mt = __ballot_sync(FULL, is_true);
    ntrue += __popc(mt);
    while (mt) {
      const int l = __ffs(mt) - 1;
      wsum = __dadd_rn(wsum, __shfl_sync(FULL, dt, l));
      mt &= mt - 1;
    }
  }
  if (lane == 0) {
    len[c] = n;
    weight[c] = wsum;
    counts[c] += ntrue;
    if (touched) touched[c] = n ? 1u : 0u;
  }
}

// Thread (class c, position j) replays the class's update list in order:
// acc += value for every listed sample with bit j set (model.cpp:54-63). In
// exact mode the element is updated in place and the class re-binarised; in
// delta mode it starts from 0.0 and only the delta is written.
template <bool DELTA>
__global__ void __launch_bounds__(256) online_update_kernel(const uint32_t* __restrict__ batch, uint32_t D, uint32_t W,
                                                            uint32_t cap, const uint32_t* __restrict__ idx,
                                                            const double* __restrict__ val,
                                                            const uint32_t* __restrict__ len,
                                                            const double* __restrict__ weight,
                                                            const uint32_t* __restrict__ tie, double* __restrict__ acc,
                                                            uint32_t* __restrict__ cv) {
  const uint32_t c = blockIdx.y;
  const uint32_t n = len[c];
  if (n == 0) return;
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  const bool valid = j < D;
  const uint32_t wi = min(j >> 5, W - 1);
  const uint32_t sh = j & 31u;
  double a = (!DELTA && valid) ? acc[static_cast<uint64_t>(c) * D + j] : 0.0;
  const uint32_t* li = idx + static_cast<uint64_t>(c) * cap;
  const double* lv = val + static_cast<uint64_t>(c) * cap;
  uint32_t k = 0;
  for (; k + 4 <= n; k += 4) {
    uint32_t wd[4];
    double v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      wd[u] = batch[static_cast<uint64_t>(li[k + u]) * W + wi];
      v[u] = lv[k + u];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if ((wd[u] >> sh) & 1u) a = __dadd_rn(a, v[u]);
    }
  }
  for (; k < n; ++k) {
    const uint32_t wd = batch[static_cast<uint64_t>(li[k]) * W + wi];
    if ((wd >> sh) & 1u) a = __dadd_rn(a, lv[k]);
  }
  if (valid) acc[static_cast<uint64_t>(c) * D + j] = a;
  if (!DELTA) {
    uint32_t bit = 0;
    if (valid) {
      const double twice = 2.0 * a;
      const double total = weight[c];
      bit = twice > total ? 1u : (twice < total ? 0u : ((tie[wi] >> sh) & 1u));
    }
    const uint32_t word = __ballot_sync(FULL, bit);
    if ((threadIdx.x & 31u) == 0 && (j >> 5) < W) cv[static_cast<uint64_t>(c) * W + (j >> 5)] = word;
  }
}

__global__ void apply_delta_scalars_kernel(uint32_t C, const double* __restrict__ dw, const uint64_t* __restrict__ dc,
                                           double* __restrict__ weight, uint64_t* __restrict__ counts) {
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  weight[c] = __dadd_rn(weight[c], dw[c]);
  counts[c] += dc[c];
}

__global__ void apply_delta_acc_kernel(uint64_t n, const double* __restrict__ d, double* __restrict__ acc) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    acc[i] = __dadd_rn(acc[i], d[i]);
  }
}

// ------------------------------------------------------ host helpers ----
unsigned sgrid(hv_context* ctx, uint64_t items, unsigned block, unsigned per_sm = 16) {
  const uint64_t want = (items + block - 1) / block;
  const uint64_t cap = static_cast<uint64_t>(ctx->sm_count) * per_sm;
  return static_cast<unsigned>(want == 0 ? 1 : std::min(want, cap));
}

// labels -> per-class histogram (validated), segment offsets and the
// class-sorted row permutation; class_rows (nullable) += histogram
void label_bucket_device(hv_context* ctx, cudaStream_t st, const int32_t* labels, size_t rows, size_t C,
                         uint32_t* hist, uint64_t* offsets, uint32_t* cursor, uint32_t* perm, uint64_t* class_rows) {
  label_hist_kernel<<<sgrid(ctx, rows, 256), 256, 0, st>>>(labels, rows, static_cast<uint32_t>(C), hist, ctx->d_err);
  launched("label_hist_kernel");
  label_scan_kernel<<<1, 32, 0, st>>>(hist, static_cast<uint32_t>(C), offsets, class_rows, cursor);
  launched("label_scan_kernel");
  label_scatter_kernel<<<sgrid(ctx, rows, 256), 256, 0, st>>>(labels, rows, static_cast<uint32_t>(C), offsets, cursor,
                                                             perm);
  launched("label_scatter_kernel");
}

// class counts of `rows` encoded rows into counts (C x 32W, added) and class_rows (added)
// (row pitch ldm words, 0 = W)
void class_counts_device(hv_context* ctx, cudaStream_t st, const uint32_t* enc, size_t rows, size_t W,
                         const int32_t* labels, size_t C, uint32_t* counts, uint64_t* class_rows, size_t ldm = 0) {
  if (rows == 0) return;
  DevBuf<uint32_t> hist(C, st), cursor(C, st), perm(rows, st);
  DevBuf<uint64_t> offsets(C + 1, st);
  hist.zero();
  label_bucket_device(ctx, st, labels, rows, C, hist.ptr, offsets.ptr, cursor.ptr, perm.ptr, class_rows);
  launch_column_count_u32(st, enc, static_cast<uint32_t>(W), perm.ptr, offsets.ptr, static_cast<uint32_t>(C), rows,
                          counts, static_cast<uint32_t>(ldm));
}

void binarize_counts_device(hv_context* ctx, cudaStream_t st, const uint32_t* counts, const uint64_t* class_rows,
                            size_t C, size_t D, const uint32_t* tie, uint32_t* cv) {
  const size_t W = words_per_row(D);
  binarize_counts_kernel<<<sgrid(ctx, C * W, 128), 128, 0, st>>>(counts, class_rows, static_cast<uint32_t>(C),
                                                                static_cast<uint32_t>(D), static_cast<uint32_t>(W), tie,
                                                                cv);
  launched("binarize_counts_kernel");
}

// (query row pitch ldq words, 0 = W; pitched rows need C < 32)
void predict_hamming_device(hv_context* ctx, cudaStream_t st, const uint32_t* cv, size_t C, size_t D,
                            const uint32_t* enc, size_t rows, int32_t* labels, double* dist, uint32_t* pops,
                            size_t ldq = 0) {
  if (rows == 0) return;
  const size_t W = words_per_row(D);
  if (ldq == 0) ldq = W;
  if (ldq < W) invalid("predict: row pitch < words per row");
  if (ldq != W) {
    if (C >= static_cast<size_t>(kScanCls)) invalid("predict: pitched query rows need fewer than 32 classes");
    const size_t W4 = (W + 3) / 4;
    const size_t smem = C * W4 * 16;
    if (C == 2 && !dist && !pops && labels && ldq % 4 == 0 && (reinterpret_cast<uintptr_t>(enc) & 15u) == 0 &&
        smem <= 96 * 1024) {
      const unsigned grid = sgrid(ctx, rows * 32, 256, 32);
      ck(cudaFuncSetAttribute(predict_two_class_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              static_cast<int>(smem)),
         "cudaFuncSetAttribute");
      predict_two_class_kernel<<<grid, 256, smem, st>>>(cv, static_cast<uint32_t>(W), static_cast<uint32_t>(ldq), enc,
                                                        rows, labels);
      launched("predict_two_class_kernel");
      return;
    }
    if (ldq % 4 == 0 && (reinterpret_cast<uintptr_t>(enc) & 15u) == 0 && smem <= 96 * 1024) {
      // 16-byte rows: class vectors staged in shared memory, uint4 row reads
      // each CTA first stages C x W4 uint4 of class vectors: fewer, longer-lived
      // CTAs amortise that for C > 2 (env HVB200_PREDICT_CTAS_PER_SM to tune)
      const char* gp = getenv("HVB200_PREDICT_CTAS_PER_SM");
      const unsigned grid = sgrid(ctx, rows * 32, 256, gp ? std::max(1, atoi(gp)) : 8);
#define HV_PP(CB)                                                                                          \
  do {                                                                                                     \
    ck(cudaFuncSetAttribute(predict_hamming_pitched_kernel<CB>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                            static_cast<int>(smem)),                                                       \
       "cudaFuncSetAttribute");                                                                            \
    predict_hamming_pitched_kernel<CB><<<grid, 256, smem, st>>>(                                           \
        cv, static_cast<uint32_t>(C), static_cast<uint32_t>(D), static_cast<uint32_t>(W),                  \
        static_cast<uint32_t>(ldq), enc, rows, labels, dist, pops);                                        \
  } while (0)
      if (C <= 2) {
        HV_PP(2);
      } else if (C <= 4) {
        HV_PP(4);
      } else if (C <= 8) {
        HV_PP(8);
      } else {
        HV_PP(16);
      }
#undef HV_PP
      launched("predict_hamming_pitched_kernel");
      return;
    }
  }
  // classes: < 32 warp per query; 32..63 CTA-tiled POPC scan; >= 64 tensor
  // cores — tcgen05 (UMMA kind::f8f6f4 on 0/2^-6 e4m3 bytes, rows in TMEM,
  // hv_predict_tc.cu) by default, the legacy mma.sync path with
  // HVB200_PREDICT_IMMA=1. Measured at 2 M rows: C = 100,
  // D = 32768: POPC 65 ms, mma.sync 27.6 ms, tcgen05 5.87 ms; C = 64,
  // D = 10000: mma.sync 7.3 ms, tcgen05 3.0 ms.
  const bool many = C >= 64 && getenv("HVB200_PREDICT_WARP") == nullptr && getenv("HVB200_PREDICT_POPC") == nullptr;
  if (many && getenv("HVB200_PREDICT_IMMA") == nullptr) {
    DevBuf<unsigned long long> best(rows, st);
    DevBuf<uint32_t> cpop(C, st);
    ck(cudaMemsetAsync(best.ptr, 0xFF, rows * sizeof(unsigned long long), st), "memset");
    class_popcount_kernel<<<grid_for(C, 8), 256, 0, st>>>(cv, static_cast<uint32_t>(C), static_cast<uint32_t>(W),
                                                          cpop.ptr);
    launched("class_popcount_kernel");
    if (!predict_tc_launch(ctx, st, cv, C, D, enc, rows, cpop.ptr, best.ptr, dist, pops)) {
      ck(cudaFuncSetAttribute(predict_imma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              static_cast<int>(kMmaSmemBytes)),
         "cudaFuncSetAttribute");
      const uint64_t items = ((rows + kMmaRows - 1) / kMmaRows) * ((C + kMmaCls - 1) / kMmaCls);
      const unsigned g = static_cast<unsigned>(std::min<uint64_t>(items, ctx->sm_count * 2ull));
      predict_imma_kernel<<<g, kMmaThreads, kMmaSmemBytes, st>>>(cv, static_cast<uint32_t>(C),
                                                                 static_cast<uint32_t>(D), static_cast<uint32_t>(W),
                                                                 enc, rows, cpop.ptr, best.ptr, dist, pops);
      launched("predict_imma_kernel");
    }
    if (labels) {
      best_to_labels_kernel<<<sgrid(ctx, rows, 256), 256, 0, st>>>(best.ptr, rows, labels);
      launched("best_to_labels_kernel");
    }
    return;
  }
  if (many) {
    DevBuf<unsigned long long> best(rows, st);
    DevBuf<uint32_t> cpop(C, st);
    ck(cudaMemsetAsync(best.ptr, 0xFF, rows * sizeof(unsigned long long), st), "memset");
    class_popcount_kernel<<<grid_for(C, 8), 256, 0, st>>>(cv, static_cast<uint32_t>(C), static_cast<uint32_t>(W),
                                                          cpop.ptr);
    launched("class_popcount_kernel");
    ck(cudaFuncSetAttribute(predict_imma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            static_cast<int>(kMmaSmemBytes)),
       "cudaFuncSetAttribute");
    int per_sm = 0;
    ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, predict_imma_kernel, kMmaThreads, kMmaSmemBytes),
       "occupancy");
    const uint64_t items = ((rows + kMmaRows - 1) / kMmaRows) * ((C + kMmaCls - 1) / kMmaCls);
    const unsigned g = static_cast<unsigned>(
        std::max<uint64_t>(1, std::min<uint64_t>(items, static_cast<uint64_t>(ctx->sm_count) * std::max(per_sm, 1))));
    predict_imma_kernel<<<g, kMmaThreads, kMmaSmemBytes, st>>>(cv, static_cast<uint32_t>(C), static_cast<uint32_t>(D),
                                                   static_cast<uint32_t>(W), enc, rows, cpop.ptr, best.ptr, dist, pops);
    launched("predict_imma_kernel");
    if (labels) {
      best_to_labels_kernel<<<sgrid(ctx, rows, 256), 256, 0, st>>>(best.ptr, rows, labels);
      launched("best_to_labels_kernel");
    }
    return;
  }
  if (C >= static_cast<size_t>(kScanCls) && getenv("HVB200_PREDICT_WARP") == nullptr) {
    DevBuf<unsigned long long> best(rows, st);
    ck(cudaMemsetAsync(best.ptr, 0xFF, rows * sizeof(unsigned long long), st), "memset");
    int per_sm = 0;
    ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, predict_tiled_kernel, 256, 0), "occupancy");
    const uint64_t items = ((rows + kScanRows - 1) / kScanRows) * ((C + kScanCls - 1) / kScanCls);
    const unsigned g = static_cast<unsigned>(
        std::max<uint64_t>(1, std::min<uint64_t>(items, static_cast<uint64_t>(ctx->sm_count) * std::max(per_sm, 1))));
    predict_tiled_kernel<<<g, 256, 0, st>>>(cv, static_cast<uint32_t>(C), static_cast<uint32_t>(D),
                                            static_cast<uint32_t>(W), enc, rows, best.ptr, dist, pops);
    launched("predict_tiled_kernel");
    if (labels) {
      best_to_labels_kernel<<<sgrid(ctx, rows, 256), 256, 0, st>>>(best.ptr, rows, labels);
      launched("best_to_labels_kernel");
    }
    return;
  }
  // 16 CTAs of 8 warps per SM (two resident waves), 4 words in flight per
  // lane per round: scripts/probe_stream.cu at CHB-MIT, 1.41 M rows — 4.11 TB/s
  // against 3.37 for one word per lane at 8 CTAs/SM and 3.84 for 10 words
  const unsigned grid = sgrid(ctx, rows * 32, 256, 16);
#define HV_PH(CB, U) \
  predict_hamming_kernel<CB, U><<<grid, 256, 0, st>>>(cv, C, D, W, ldq, enc, rows, labels, dist, pops)
#define HV_PH_U(CB) \
  if (W <= 64) {    \
    HV_PH(CB, 2);   \
  } else {          \
    HV_PH(CB, 4);   \
  }
  if (C <= 2) {
    HV_PH_U(2)
  } else if (C <= 4) {
    HV_PH_U(4)
  } else if (C <= 8) {
    HV_PH_U(8)
  } else {
    HV_PH_U(16)
  }
#undef HV_PH_U
#undef HV_PH
  launched("predict_hamming_kernel");
}

void cosine_scores_device(hv_context* ctx, cudaStream_t st, const double* acc, size_t C, size_t D, const uint32_t* enc,
                          size_t rows, double* scores, uint64_t err_base) {
  const size_t W = words_per_row(D);
  DevBuf<double> norm(C, st);
  class_norms_kernel<<<grid_for(C, 64), 64, 0, st>>>(acc, C, D, norm.ptr);
  launched("class_norms_kernel");
  if (rows == 0) return;
  cosine_scores_kernel<<<sgrid(ctx, rows * C, 128, 64), 128, 0, st>>>(acc, norm.ptr, C, D, W, enc, rows, scores,
                                                                      ctx->d_err, err_base);
  launched("cosine_scores_kernel");
}

void refresh_device(hv_context* ctx, cudaStream_t st, const double* acc, const double* weight, const uint32_t* touched,
                    size_t C, size_t D, const uint32_t* tie, uint32_t* cv) {
  const size_t W = words_per_row(D);
  refresh_kernel<<<sgrid(ctx, C * W * 32, 256), 256, 0, st>>>(acc, weight, touched, C, D, W, tie, cv);
  launched("refresh_kernel");
}

// Scratch for one online batch.
struct OnlineScratch {
  DevBuf<int32_t> pred;
  DevBuf<double> dtrue, pen, val, scores;
  DevBuf<uint32_t> idx, len;
  size_t cap;
  OnlineScratch(size_t C, size_t cap_, bool cosine, cudaStream_t st)
      : pred(cap_, st), dtrue(cap_, st), pen(cap_, st), val(C * cap_, st), scores(cosine ? C * cap_ : 0, st),
        idx(C * cap_, st), len(C, st), cap(cap_) {}
};

// One online batch (exact or delta) on device-resident state.
template <bool DELTA>
void online_batch(hv_context* ctx, cudaStream_t st, OnlineScratch& s, hv_metric metric, const uint32_t* snap_cv,
                  const double* snap_acc, size_t C, size_t D, const uint32_t* batch, size_t rows, const int32_t* labels,
                  double gamma, const uint32_t* tie, double* acc, double* weight, uint64_t* counts, uint32_t* cv,
                  uint32_t* touched) {
  if (rows == 0) return;
  const size_t W = words_per_row(D);
  if (metric == HV_METRIC_HAMMING) {
    online_score_hamming_kernel<<<sgrid(ctx, rows * 32, 256, 8), 256, 0, st>>>(
        snap_cv, C, D, W, batch, rows, labels, gamma, s.pred.ptr, s.dtrue.ptr, s.pen.ptr);
    launched("online_score_hamming_kernel");
  } else {
    cosine_scores_device(ctx, st, snap_acc, C, D, batch, rows, s.scores.ptr, 0);
    online_score_cosine_kernel<<<sgrid(ctx, rows, 128), 128, 0, st>>>(s.scores.ptr, C, rows, labels, gamma, s.pred.ptr,
                                                                      s.dtrue.ptr, s.pen.ptr);
    launched("online_score_cosine_kernel");
  }
  online_lists_kernel<<<C, 32, 0, st>>>(labels, s.pred.ptr, s.dtrue.ptr, s.pen.ptr, rows, C, s.cap, s.idx.ptr,
                                        s.val.ptr, s.len.ptr, weight, counts, touched);
  launched("online_lists_kernel");
  dim3 grid((D + 255) / 256, C);
  online_update_kernel<DELTA><<<grid, 256, 0, st>>>(batch, D, W, s.cap, s.idx.ptr, s.val.ptr, s.len.ptr, weight, tie,
                                                    acc, cv);
  launched("online_update_kernel");
}

void train_online_device(hv_context* ctx, cudaStream_t st, hv_metric metric, const uint32_t* enc, size_t rows, size_t D,
                         const int32_t* labels, size_t C, size_t bsz, double gamma, const uint32_t* tie, double* acc,
                         double* weight, uint64_t* counts, uint32_t* cv) {
  const size_t W = words_per_row(D);
  const size_t first = std::min(bsz, rows);
  {
    DevBuf<uint32_t> cnt(C * 32 * W, st);
    DevBuf<uint64_t> crow(C, st);
    cnt.zero();
    crow.zero();
    class_counts_device(ctx, st, enc, first, W, labels, C, cnt.ptr, crow.ptr);
    init_from_counts_kernel<<<sgrid(ctx, C * D, 256), 256, 0, st>>>(cnt.ptr, crow.ptr, C, D, W, acc, weight, counts);
    launched("init_from_counts_kernel");
    binarize_counts_device(ctx, st, cnt.ptr, crow.ptr, C, D, tie, cv);
  }
  if (rows == 0) return;
  const char* legacy = getenv("HVB200_ONLINE_LEGACY");
  if (metric == HV_METRIC_HAMMING && !(legacy && legacy[0] == '1')) {
    train_online_persistent(ctx, st, enc, rows, D, labels, C, bsz, gamma, tie, acc, weight, counts, cv);
    return;
  }
  OnlineScratch s(C, std::min(bsz, rows), metric == HV_METRIC_COSINE, st);
  DevBuf<double> snap(metric == HV_METRIC_COSINE ? C * D : 0, st);
  for (size_t start = 0; start < rows; start += bsz) {
    const size_t n = std::min(bsz, rows - start);
    const double* snap_acc = nullptr;
    if (metric == HV_METRIC_COSINE) {
      ck(cudaMemcpyAsync(snap.ptr, acc, C * D * sizeof(double), cudaMemcpyDeviceToDevice, st), "snapshot");
      snap_acc = snap.ptr;
    }
    // The class vectors are only rewritten by the update kernel after every
    // score of this batch has been computed, so `cv` itself is the snapshot.
    online_batch<false>(ctx, st, s, metric, cv, snap_acc, C, D, enc + start * W, n, labels + start, gamma, tie, acc,
                        weight, counts, cv, nullptr);
  }
}

void check_labels_host(const int32_t* labels, size_t n_labels, size_t rows, size_t C, const char* who) {
  if (n_labels != rows) {
    invalid(std::string(who) + ": " + std::to_string(n_labels) + " labels for " + std::to_string(rows) + " rows");
  }
  for (size_t i = 0; i < n_labels; ++i) {
    if (labels[i] < 0 || static_cast<size_t>(labels[i]) >= C) {
      invalid(std::string(who) + ": label " + std::to_string(labels[i]) + " at row " + std::to_string(i) +
              " out of range (classes = " + std::to_string(C) + ")");
    }
  }
}

void check_model_config(const hv_model* m) {
  if (m == nullptr) invalid("null hv_model");
  if (m->class_count == 0) invalid("make_empty_model: need at least one class");
  if (m->dim == 0) invalid("make_empty_model: dim must be >= 1");
  if (m->gamma < 0.0) invalid("make_empty_model: gamma must be >= 0");
  if (m->metric != HV_METRIC_HAMMING && m->metric != HV_METRIC_COSINE) fail(HV_ERR_LOGIC, "bad Metric");
}

// Device copy of a host hv_model's arrays.
struct DevModel {
  DevBuf<double> acc, weight;
  DevBuf<uint64_t> counts;
  DevBuf<uint32_t> cv, tie;
  DevModel(const hv_model* m, cudaStream_t st, bool upload)
      : acc(m->class_count * m->dim, st), weight(m->class_count, st), counts(m->class_count, st),
        cv(m->class_count * words_per_row(m->dim), st), tie(words_per_row(m->dim), st) {
    if (upload) {
      acc.upload(m->accumulators);
      weight.upload(m->class_weight);
      counts.upload(m->sample_counts);
      cv.upload(m->class_vectors);
    }
    tie.upload(m->tiebreak);
  }
  void download(hv_model* m) {
    acc.download(m->accumulators);
    weight.download(m->class_weight);
    counts.download(m->sample_counts);
    cv.download(m->class_vectors);
  }
};

void fill_tiebreak(hv_model* m) { generate_random_words(1, m->dim, derive_seed(m->seed, 3), m->tiebreak); }

}  // namespace hvb

using namespace hvb;

extern "C" {

hv_status hv_make_empty_model(hv_model* m) {
  return guarded([&] {
    check_model_config(m);
    const size_t C = m->class_count, D = m->dim, W = words_per_row(D);
    std::fill(m->accumulators, m->accumulators + C * D, 0.0);
    std::fill(m->class_weight, m->class_weight + C, 0.0);
    std::fill(m->sample_counts, m->sample_counts + C, 0ull);
    fill_tiebreak(m);
    for (size_t c = 0; c < C; ++c) std::copy(m->tiebreak, m->tiebreak + W, m->class_vectors + c * W);
  });
}

// model.cpp:169-181 hamming_distance(_words): popc(a ^ b) / dim in double, the
// same one-row Hamming scan as predict (class = b, query = a).
hv_status hv_hamming_distance(hv_context* ctx, const uint32_t* a, const uint32_t* b, size_t dim, double* out) {
  return guarded([&] {
    require(ctx);
    if (dim == 0) invalid("hamming_distance: dim must be >= 1");
    const size_t W = words_per_row(dim);
    cudaStream_t st = ctx->stream;
    DevBuf<uint32_t> da(W, st), db(W, st);
    DevBuf<double> dd(1, st);
    da.upload(a);
    db.upload(b);
    predict_hamming_device(ctx, st, db.ptr, 1, dim, da.ptr, 1, nullptr, dd.ptr, nullptr);
    dd.download(out);
    sync(ctx);
  });
}

// model.cpp:183-196 cosine_similarity: dot(acc, row) / (|acc| sqrt(popc(row))),
// sequential fp64 like the reference; a zero accumulator or an empty row is
// a domain error.
hv_status hv_cosine_similarity(hv_context* ctx, const double* acc, size_t acc_len, const uint32_t* row, size_t dim,
                               double* out) {
  return guarded([&] {
    require(ctx);
    if (acc_len != dim) invalid("cosine_similarity: accumulator length != dim");
    if (dim == 0) invalid("cosine_similarity: dim must be >= 1");
    const size_t W = words_per_row(dim);
    cudaStream_t st = ctx->stream;
    DevBuf<double> dacc(dim, st), dd(1, st);
    DevBuf<uint32_t> dr(W, st);
    dacc.upload(acc);
    dr.upload(row);
    cosine_scores_device(ctx, st, dacc.ptr, 1, dim, dr.ptr, 1, dd.ptr, 0);
    dd.download(out);
    sync(ctx);
    unsigned long long l[kErrKinds];
    read_latch(ctx, l);
    if (l[kErrZeroQuery] != ~0ull || std::isinf(*out)) {
      reset_latch(ctx);
      fail(HV_ERR_DOMAIN, "cosine_similarity: zero vector");
    }
  });
}

hv_status hv_refresh_binarization(hv_context* ctx, hv_model* m, size_t class_index) {
  return guarded([&] {
    require(ctx);
    check_model_config(m);
    const size_t C = m->class_count;
    if (class_index != SIZE_MAX && class_index >= C) invalid("refresh_binarization: class index out of range");
    DevModel dm(m, ctx->stream, true);
    DevBuf<uint32_t> touched(C, ctx->stream);
    std::vector<uint32_t> t(C, class_index == SIZE_MAX ? 1u : 0u);
    if (class_index != SIZE_MAX) t[class_index] = 1u;
    touched.upload(t.data());
    refresh_device(ctx, ctx->stream, dm.acc.ptr, dm.weight.ptr, touched.ptr, C, m->dim, dm.tie.ptr, dm.cv.ptr);
    dm.cv.download(m->class_vectors);
    sync(ctx);
  });
}

hv_status hv_train_classical(hv_context* ctx, const uint32_t* encoded, size_t rows, size_t dim, const int32_t* labels,
                             size_t n_labels, hv_model* m) {
  return guarded([&] {
    require(ctx);
    if (m == nullptr) invalid("null hv_model");
    check_labels_host(labels, n_labels, rows, m->class_count, "train_classical");
    m->dim = dim;
    check_model_config(m);
    fill_tiebreak(m);
    const size_t C = m->class_count, W = words_per_row(dim);
    cudaStream_t st = ctx->stream;
    DevBuf<uint32_t> enc(rows * W, st), cnt(C * 32 * W, st), cv(C * W, st), tie(W, st);
    DevBuf<int32_t> y(rows, st);
    DevBuf<uint64_t> crow(C, st);
    enc.upload(encoded);
    y.upload(labels);
    tie.upload(m->tiebreak);
    cnt.zero();
    crow.zero();
    class_counts_device(ctx, st, enc.ptr, rows, W, y.ptr, C, cnt.ptr, crow.ptr);
    binarize_counts_device(ctx, st, cnt.ptr, crow.ptr, C, dim, tie.ptr, cv.ptr);
    std::vector<uint32_t> hc(C * 32 * W);
    cnt.download(hc.data());
    crow.download(m->sample_counts);
    cv.download(m->class_vectors);
    sync(ctx);
    for (size_t c = 0; c < C; ++c) {
      m->class_weight[c] = static_cast<double>(m->sample_counts[c]);
      for (size_t j = 0; j < dim; ++j) m->accumulators[c * dim + j] = static_cast<double>(hc[c * 32 * W + j]);
    }
  });
}

hv_status hv_online_update(hv_context* ctx, hv_model* m, const uint32_t* batch, size_t rows, size_t dim,
                           const int32_t* labels, size_t n_labels, const uint32_t* snap_cv, const double* snap_acc) {
  return guarded([&] {
    require(ctx);
    check_model_config(m);
    if (dim != m->dim) invalid("online_update: batch dim != model dim");
    check_labels_host(labels, n_labels, rows, m->class_count, "online_update");
    if (rows == 0) return;
    if (m->metric == HV_METRIC_COSINE && snap_acc == nullptr) invalid("online_update: cosine needs snapshot accumulators");
    const size_t C = m->class_count, D = m->dim, W = words_per_row(D);
    cudaStream_t st = ctx->stream;
    DevModel dm(m, st, true);
    DevBuf<uint32_t> b(rows * W, st), scv(C * W, st);
    DevBuf<int32_t> y(rows, st);
    DevBuf<double> sacc(m->metric == HV_METRIC_COSINE ? C * D : 0, st);
    b.upload(batch);
    y.upload(labels);
    scv.upload(snap_cv);
    if (m->metric == HV_METRIC_COSINE) sacc.upload(snap_acc);
    OnlineScratch s(C, rows, m->metric == HV_METRIC_COSINE, st);
    online_batch<false>(ctx, st, s, m->metric, scv.ptr, sacc.ptr, C, D, b.ptr, rows, y.ptr, m->gamma, dm.tie.ptr,
                        dm.acc.ptr, dm.weight.ptr, dm.counts.ptr, dm.cv.ptr, nullptr);
    dm.download(m);
    unsigned long long l[kErrKinds];
    read_latch(ctx, l);
    if (l[kErrZeroQuery] != ~0ull) {
      reset_latch(ctx);
      fail(HV_ERR_DOMAIN, "cosine_similarity: zero query vector");
    }
  });
}

hv_status hv_train_online(hv_context* ctx, const uint32_t* encoded, size_t rows, size_t dim, const int32_t* labels,
                          size_t n_labels, size_t batch_size, hv_model* m) {
  return guarded([&] {
    require(ctx);
    if (batch_size == 0) invalid("train_online: batch_size must be >= 1");
    if (m == nullptr) invalid("null hv_model");
    if (n_labels != rows) {
      invalid("train_online: " + std::to_string(n_labels) + " labels for " + std::to_string(rows) + " rows");
    }
    const size_t first = std::min(batch_size, rows);
    check_labels_host(labels, first, first, m->class_count, "train_classical");
    m->dim = dim;
    check_model_config(m);
    for (size_t start = 0; start < rows; start += batch_size) {
      const size_t n = std::min(batch_size, rows - start);
      check_labels_host(labels + start, n, n, m->class_count, "online_update");
    }
    fill_tiebreak(m);
    const size_t C = m->class_count, W = words_per_row(dim);
    cudaStream_t st = ctx->stream;
    DevModel dm(m, st, false);
    DevBuf<uint32_t> enc(rows * W, st);
    DevBuf<int32_t> y(rows, st);
    enc.upload(encoded);
    y.upload(labels);
    train_online_device(ctx, st, m->metric, enc.ptr, rows, dim, y.ptr, C, batch_size, m->gamma, dm.tie.ptr, dm.acc.ptr,
                        dm.weight.ptr, dm.counts.ptr, dm.cv.ptr);
    dm.download(m);
    unsigned long long l[kErrKinds];
    read_latch(ctx, l);
    if (l[kErrZeroQuery] != ~0ull) {
      reset_latch(ctx);
      fail(HV_ERR_DOMAIN, "cosine_similarity: zero query vector");
    }
  });
}

hv_status hv_predict(hv_context* ctx, const hv_model* m, const uint32_t* encoded, size_t rows, size_t dim,
                     int32_t* labels_out, double* distances_out) {
  return guarded([&] {
    require(ctx);
    check_model_config(m);
    if (dim != m->dim) invalid("predict: query dim != model dim");
    if (rows == 0) return;
    const size_t C = m->class_count, D = m->dim, W = words_per_row(D);
    cudaStream_t streams[2] = {ctx->stream, ctx->aux};
    DevBuf<uint32_t> cv(C * W, ctx->stream);
    DevBuf<double> acc(m->metric == HV_METRIC_COSINE ? C * D : 0, ctx->stream);
    cv.upload(m->class_vectors);
    if (m->metric == HV_METRIC_COSINE) acc.upload(m->accumulators);
    sync(ctx);
    // double-buffered chunks: H2D(k+1) / D2H(k-1) overlap the scan of chunk k
    const size_t chunk = std::max<size_t>(1, std::min<size_t>(rows, (size_t(64) << 20) / (W * 4)));
    DevBuf<uint32_t> q[2] = {DevBuf<uint32_t>(chunk * W, ctx->stream), DevBuf<uint32_t>(chunk * W, ctx->stream)};
    DevBuf<int32_t> lab[2] = {DevBuf<int32_t>(chunk, ctx->stream), DevBuf<int32_t>(chunk, ctx->stream)};
    const bool want_d = distances_out != nullptr || m->metric == HV_METRIC_COSINE;
    DevBuf<double> dist[2] = {DevBuf<double>(want_d ? chunk * C : 0, ctx->stream),
                              DevBuf<double>(want_d ? chunk * C : 0, ctx->stream)};
    sync(ctx);
    size_t k = 0;
    for (size_t r0 = 0; r0 < rows; r0 += chunk, ++k) {
      const size_t n = std::min(chunk, rows - r0);
      cudaStream_t st = streams[k & 1];
      const int b = static_cast<int>(k & 1);
      ck(cudaMemcpyAsync(q[b].ptr, encoded + r0 * W, n * W * 4, cudaMemcpyHostToDevice, st), "H2D queries");
      if (m->metric == HV_METRIC_HAMMING) {
        predict_hamming_device(ctx, st, cv.ptr, C, D, q[b].ptr, n, lab[b].ptr, want_d ? dist[b].ptr : nullptr, nullptr);
      } else {
        cosine_scores_device(ctx, st, acc.ptr, C, D, q[b].ptr, n, dist[b].ptr, r0);
        argmax_kernel<<<sgrid(ctx, n, 128), 128, 0, st>>>(dist[b].ptr, n, C, lab[b].ptr);
        launched("argmax_kernel");
      }
      ck(cudaMemcpyAsync(labels_out + r0, lab[b].ptr, n * 4, cudaMemcpyDeviceToHost, st), "D2H labels");
      if (distances_out) {
        ck(cudaMemcpyAsync(distances_out + r0 * C, dist[b].ptr, n * C * 8, cudaMemcpyDeviceToHost, st), "D2H dist");
      }
    }
    ck(cudaStreamSynchronize(ctx->aux), "sync aux");
    sync(ctx);
    unsigned long long l[kErrKinds];
    read_latch(ctx, l);
    if (l[kErrZeroQuery] != ~0ull) {
      reset_latch(ctx);
      fail(HV_ERR_DOMAIN, "cosine_similarity: zero query vector");
    }
  });
}

// ------------------------------------------------------- device API ----
hv_status hv_dev_class_counts(hv_context* ctx, const uint32_t* encoded, size_t rows, size_t dim, const int32_t* labels,
                              size_t class_count, uint32_t* counts, uint64_t* class_rows) {
  return guarded([&] {
    require(ctx);
    if (class_count == 0) invalid("class_counts: need at least one class");
    class_counts_device(ctx, ctx->stream, encoded, rows, words_per_row(dim), labels, class_count, counts, class_rows);
  });
}

hv_status hv_dev_class_counts_pitched(hv_context* ctx, const uint32_t* encoded, size_t ldw, size_t rows, size_t dim,
                                      const int32_t* labels, size_t class_count, uint32_t* counts,
                                      uint64_t* class_rows) {
  return guarded([&] {
    require(ctx);
    if (class_count == 0) invalid("class_counts: need at least one class");
    class_counts_device(ctx, ctx->stream, encoded, rows, words_per_row(dim), labels, class_count, counts, class_rows,
                        ldw);
  });
}

size_t hv_row_pitch_words(size_t dim) { return (words_per_row(dim) + 3) / 4 * 4; }

hv_status hv_dev_binarize_counts(hv_context* ctx, const uint32_t* counts, const uint64_t* class_rows, size_t class_count,
                                 size_t dim, const uint32_t* tiebreak, uint32_t* class_vectors) {
  return guarded([&] {
    require(ctx);
    binarize_counts_device(ctx, ctx->stream, counts, class_rows, class_count, dim, tiebreak, class_vectors);
  });
}

hv_status hv_dev_predict_hamming(hv_context* ctx, const uint32_t* class_vectors, size_t class_count, size_t dim,
                                 const uint32_t* encoded, size_t rows, int32_t* labels, double* distances,
                                 uint32_t* popcounts) {
  return guarded([&] {
    require(ctx);
    if (class_count == 0 || dim == 0) invalid("predict: empty model");
    predict_hamming_device(ctx, ctx->stream, class_vectors, class_count, dim, encoded, rows, labels, distances,
                           popcounts);
  });
}

hv_status hv_dev_predict_hamming_pitched(hv_context* ctx, const uint32_t* class_vectors, size_t class_count,
                                         size_t dim, const uint32_t* encoded, size_t ldw, size_t rows, int32_t* labels,
                                         double* distances, uint32_t* popcounts) {
  return guarded([&] {
    require(ctx);
    if (class_count == 0 || dim == 0) invalid("predict: empty model");
    predict_hamming_device(ctx, ctx->stream, class_vectors, class_count, dim, encoded, rows, labels, distances,
                           popcounts, ldw);
  });
}

hv_status hv_dev_train_online(hv_context* ctx, const uint32_t* encoded, size_t rows, size_t dim, const int32_t* labels,
                              size_t class_count, size_t batch_size, double gamma, const uint32_t* tiebreak,
                              double* acc, double* weight, uint64_t* counts, uint32_t* class_vectors) {
  return guarded([&] {
    require(ctx);
    if (batch_size == 0) invalid("train_online: batch_size must be >= 1");
    if (class_count == 0 || dim == 0) invalid("train_online: empty model");
    train_online_device(ctx, ctx->stream, HV_METRIC_HAMMING, encoded, rows, dim, labels, class_count, batch_size, gamma,
                        tiebreak, acc, weight, counts, class_vectors);
  });
}

hv_status hv_dev_online_delta(hv_context* ctx, const uint32_t* class_vectors, size_t class_count, size_t dim,
                              const uint32_t* batch, size_t rows, const int32_t* labels, double gamma,
                              double* delta_acc, double* delta_weight, uint64_t* delta_counts,
                              uint32_t* delta_touched) {
  return guarded([&] {
    require(ctx);
    cudaStream_t st = ctx->stream;
    const size_t C = class_count, D = dim;
    ck(cudaMemsetAsync(delta_acc, 0, C * D * sizeof(double), st), "memset");
    ck(cudaMemsetAsync(delta_weight, 0, C * sizeof(double), st), "memset");
    ck(cudaMemsetAsync(delta_counts, 0, C * sizeof(uint64_t), st), "memset");
    ck(cudaMemsetAsync(delta_touched, 0, C * sizeof(uint32_t), st), "memset");
    if (rows == 0) return;
    OnlineScratch s(C, rows, false, st);
    online_batch<true>(ctx, st, s, HV_METRIC_HAMMING, class_vectors, nullptr, C, D, batch, rows, labels, gamma, nullptr,
                       delta_acc, delta_weight, delta_counts, nullptr, delta_touched);
  });
}

// ---- D-sliced exact online training (one word slice per rank) ----
hv_status hv_dev_online_slice_init(hv_context* ctx, const uint32_t* batch0, size_t rows0, const int32_t* labels,
                                   size_t class_count, size_t dim, size_t word_begin, size_t words,
                                   const uint32_t* tiebreak, double* acc, double* weight, uint64_t* counts,
                                   uint32_t* class_vectors) {
  return guarded([&] {
    require(ctx);
    cudaStream_t st = ctx->stream;
    const size_t C = class_count, W = words_per_row(dim);
    if (C == 0 || dim == 0) invalid("train_online: empty model");
    if (words == 0 || word_begin + words > W) invalid("online slice: word range outside the row");
    const size_t Ds = std::min(dim, 32 * (word_begin + words)) - 32 * word_begin;
    DevBuf<uint32_t> cnt(C * 32 * words, st);
    DevBuf<uint64_t> crow(C, st);
    cnt.zero();
    crow.zero();
    class_counts_device(ctx, st, batch0, rows0, words, labels, C, cnt.ptr, crow.ptr);
    init_from_counts_kernel<<<sgrid(ctx, C * Ds, 256), 256, 0, st>>>(cnt.ptr, crow.ptr, C, Ds, words, acc, weight,
                                                                      counts);
    launched("init_from_counts_kernel");
    binarize_counts_device(ctx, st, cnt.ptr, crow.ptr, C, Ds, tiebreak + word_begin, class_vectors);
  });
}

hv_status hv_dev_online_partial_popc(hv_context* ctx, const uint32_t* class_vectors, size_t class_count, size_t words,
                                     const uint32_t* batch, size_t rows, uint32_t* popc) {
  return guarded([&] {
    require(ctx);
    if (rows == 0 || class_count == 0) return;
    online_partial_popc_kernel<<<sgrid(ctx, rows * 32, 256, 8), 256, 0, ctx->stream>>>(
        class_vectors, static_cast<uint32_t>(class_count), static_cast<uint32_t>(words), batch, rows, popc, nullptr,
        0u);
    launched("online_partial_popc_kernel");
  });
}

hv_status hv_dev_online_partial_popc_peers(hv_context* ctx, const uint32_t* class_vectors, size_t class_count,
                                           size_t words, const uint32_t* batch, size_t rows,
                                           uint32_t* const* peer_popc, size_t world) {
  return guarded([&] {
    require(ctx);
    if (world == 0 || world > 64) invalid("online_partial_popc_peers: world must be 1..64");
    if (rows == 0 || class_count == 0) return;
    online_partial_popc_kernel<<<sgrid(ctx, rows * 32, 256, 8), 256, 0, ctx->stream>>>(
        class_vectors, static_cast<uint32_t>(class_count), static_cast<uint32_t>(words), batch, rows, nullptr,
        peer_popc, static_cast<uint32_t>(world));
    launched("online_partial_popc_kernel");
  });
}

hv_status hv_dev_online_slice_update(hv_context* ctx, const uint32_t* popc, size_t class_count, size_t dim,
                                     size_t word_begin, size_t words, const uint32_t* batch, size_t rows,
                                     const int32_t* labels, double gamma, const uint32_t* tiebreak, double* acc,
                                     double* weight, uint64_t* counts, uint32_t* class_vectors) {
  return guarded([&] {
    require(ctx);
    cudaStream_t st = ctx->stream;
    const size_t C = class_count, W = words_per_row(dim);
    if (words == 0 || word_begin + words > W) invalid("online slice: word range outside the row");
    if (rows == 0) return;
    const size_t Ds = std::min(dim, 32 * (word_begin + words)) - 32 * word_begin;
    OnlineScratch s(C, rows, false, st);
    online_score_popc_kernel<<<sgrid(ctx, rows, 128), 128, 0, st>>>(popc, static_cast<uint32_t>(C),
                                                                    static_cast<uint32_t>(dim), rows, labels, gamma,
                                                                    s.pred.ptr, s.dtrue.ptr, s.pen.ptr, ctx->d_err);
    launched("online_score_popc_kernel");
    online_lists_kernel<<<C, 32, 0, st>>>(labels, s.pred.ptr, s.dtrue.ptr, s.pen.ptr, rows, C, s.cap, s.idx.ptr,
                                          s.val.ptr, s.len.ptr, weight, counts, nullptr);
    launched("online_lists_kernel");
    dim3 grid((Ds + 255) / 256, C);
    online_update_kernel<false><<<grid, 256, 0, st>>>(batch, Ds, words, s.cap, s.idx.ptr, s.val.ptr, s.len.ptr, weight,
                                                      tiebreak + word_begin, acc, class_vectors);
    launched("online_update_kernel");
  });
}

// All batches of the word-sliced exact online mode with the popcount exchange
// fused over peer memory, enqueued from here in one call (per batch: partial
// popcounts added into every rank's parity slot, signal, wait, score, lists,
// slice update, slot reset) — no host round trip and no per-batch allocation.
// Epochs epoch0 + 1 .. epoch0 + nbatches are used; they must exceed every
// epoch already signalled on these buffers.
hv_status hv_dev_online_sliced_run_peers(hv_context* ctx, const uint32_t* enc_slice, size_t rows, size_t words,
                                         size_t word_begin, size_t dim, const int32_t* labels, size_t class_count,
                                         size_t batch_size, double gamma, const uint32_t* tiebreak,
                                         uint32_t* const* peer_popc0, uint32_t* const* peer_popc1, uint32_t* own_popc0,
                                         uint32_t* own_popc1, uint32_t* const* peer_flags, const uint32_t* own_flags,
                                         size_t world, size_t rank, uint32_t epoch0, double* acc, double* weight,
                                         uint64_t* counts, uint32_t* class_vectors) {
  return guarded([&] {
    require(ctx);
    cudaStream_t st = ctx->stream;
    const size_t C = class_count, W = words_per_row(dim);
    if (C == 0 || dim == 0) invalid("train_online: empty model");
    if (batch_size == 0) invalid("train_online: batch_size must be >= 1");
    if (words == 0 || word_begin + words > W) invalid("online slice: word range outside the row");
    if (world == 0 || world > 64 || rank >= world) invalid("online_sliced_run_peers: bad world/rank");
    if (rows == 0) return;
    const size_t Ds = std::min(dim, 32 * (word_begin + words)) - 32 * word_begin;
    const size_t cap = std::min(batch_size, rows);
    OnlineScratch s(C, cap, false, st);
    uint32_t ep = epoch0;
    for (size_t b0 = 0; b0 < rows; b0 += batch_size) {
      const size_t n = std::min(batch_size, rows - b0);
      ++ep;
      const bool odd = ep & 1u;
      uint32_t* const* peers = odd ? peer_popc1 : peer_popc0;
      uint32_t* own = odd ? own_popc1 : own_popc0;
      const uint32_t* batch = enc_slice + b0 * words;
      online_partial_popc_kernel<<<sgrid(ctx, n * 32, 256, 8), 256, 0, st>>>(
          class_vectors, static_cast<uint32_t>(C), static_cast<uint32_t>(words), batch, n, nullptr, peers,
          static_cast<uint32_t>(world));
      launched("online_partial_popc_kernel");
      if (hv_dev_signal_peers(ctx, peer_flags, world, rank, ep) != HV_OK) fail(HV_ERR_CUDA, hv_last_error());
      if (hv_dev_wait_peers(ctx, own_flags, world, ep) != HV_OK) fail(HV_ERR_CUDA, hv_last_error());
      online_score_popc_kernel<<<sgrid(ctx, n, 128), 128, 0, st>>>(own, static_cast<uint32_t>(C),
                                                                  static_cast<uint32_t>(dim), n, labels + b0, gamma,
                                                                  s.pred.ptr, s.dtrue.ptr, s.pen.ptr, ctx->d_err);
      launched("online_score_popc_kernel");
      online_lists_kernel<<<C, 32, 0, st>>>(labels + b0, s.pred.ptr, s.dtrue.ptr, s.pen.ptr, n, C, s.cap, s.idx.ptr,
                                            s.val.ptr, s.len.ptr, weight, counts, nullptr);
      launched("online_lists_kernel");
      dim3 grid((Ds + 255) / 256, C);
      online_update_kernel<false><<<grid, 256, 0, st>>>(batch, Ds, words, s.cap, s.idx.ptr, s.val.ptr, s.len.ptr,
                                                        weight, tiebreak + word_begin, acc, class_vectors);
      launched("online_update_kernel");
      ck(cudaMemsetAsync(own, 0, n * C * sizeof(uint32_t), st), "reset popcount slot");
    }
    unsigned long long l[kErrKinds];
    sync(ctx);
    read_latch(ctx, l);
    if (l[kErrLabel] != ~0ull) {
      reset_latch(ctx);
      invalid("online_update: label out of range at batch row " + std::to_string(l[kErrLabel]));
    }
  });
}

hv_status hv_dev_apply_online_delta(hv_context* ctx, size_t class_count, size_t dim, const double* delta_acc,
                                    const double* delta_weight, const uint64_t* delta_counts, const uint32_t* touched,
                                    const uint32_t* tiebreak, double* acc, double* weight, uint64_t* counts,
                                    uint32_t* class_vectors) {
  return guarded([&] {
    require(ctx);
    cudaStream_t st = ctx->stream;
    const size_t C = class_count, D = dim;
    apply_delta_scalars_kernel<<<grid_for(C, 64), 64, 0, st>>>(C, delta_weight, delta_counts, weight, counts);
    launched("apply_delta_scalars_kernel");
    apply_delta_acc_kernel<<<sgrid(ctx, C * D, 256), 256, 0, st>>>(C * D, delta_acc, acc);
    launched("apply_delta_acc_kernel");
    refresh_device(ctx, st, acc, weight, touched, C, D, tiebreak, class_vectors);
  });
}

}  // extern "C"

// ------------------------------------------------------------- fold ----
// experiment.cpp:159-177 with HBM-resident hypervectors.
struct hv_fold {
  size_t train_rows = 0, test_rows = 0, F = 0, D = 0, W = 0, C = 0;
  size_t ldw = 0;  // row pitch of enc: W rounded up to 16 bytes (uint4 / TMA row reads)
  hvb::DevBuf<uint32_t> enc, counts;
  hvb::DevBuf<uint64_t> class_rows;
};

struct hv_dataset {
  size_t rows = 0, F = 0;
  hvb::DevBuf<double> X;
  hvb::DevBuf<int32_t> y;
};

namespace hvb {
namespace {

__global__ void gather_labels_kernel(const int32_t* __restrict__ y, const uint64_t* __restrict__ idx, uint64_t n,
                                     int32_t* __restrict__ out) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    out[i] = y[idx[i]];
  }
}

// validates labels into the label latch (first offending index)
void check_labels_device(hv_context* ctx, cudaStream_t st, const int32_t* y, size_t n, size_t C) {
  if (n == 0) return;
  DevBuf<uint32_t> hist(C, st);
  hist.zero();
  label_hist_kernel<<<sgrid(ctx, n, 256), 256, 0, st>>>(y, n, static_cast<uint32_t>(C), hist.ptr, ctx->d_err);
  launched("label_hist_kernel");
}

void check_indices(const uint64_t* idx, size_t n, size_t rows, const char* what) {
  for (size_t i = 0; i < n; ++i) {
    if (idx[i] >= rows) {
      invalid(std::string("dataset_fold: ") + what + " row index " + std::to_string(idx[i]) + " out of range (rows = " +
              std::to_string(rows) + ")");
    }
  }
}

}  // namespace
}  // namespace hvb

extern "C" {

hv_status hv_fold_encode_train(hv_context* ctx, const uint32_t* train_bins, size_t train_rows,
                               const int32_t* train_labels, const uint32_t* test_bins, size_t test_rows,
                               size_t features, const uint32_t* id_vectors, const uint32_t* value_vectors,
                               size_t bins, size_t dim, const uint32_t* encode_tiebreak, size_t class_count,
                               hv_fold** out) {
  return guarded([&] {
    require(ctx);
    if (!out) invalid("fold: null output");
    *out = nullptr;
    if (features == 0 || dim == 0 || class_count == 0) invalid("fold: features, dim and classes must be >= 1");
    auto fold = std::make_unique<hv_fold>();
    const size_t W = words_per_row(dim), ldb = bins_pitch(features), rows = train_rows + test_rows;
    fold->train_rows = train_rows;
    fold->test_rows = test_rows;
    fold->F = features;
    fold->D = dim;
    fold->W = W;
    fold->C = class_count;
    fold->ldw = hv_row_pitch_words(dim);
    const size_t ldw = fold->ldw;
    cudaStream_t st = ctx->stream;
    fold->enc = DevBuf<uint32_t>(rows * ldw, st);
    fold->counts = DevBuf<uint32_t>(class_count * 32 * W, st);
    fold->class_rows = DevBuf<uint64_t>(class_count, st);
    fold->counts.zero();
    fold->class_rows.zero();
    DevBuf<uint32_t> d_id(features * W, st), d_val(bins * W, st), d_tie(W, st);
    DevBuf<int32_t> d_y(train_rows, st);
    d_id.upload(id_vectors);
    d_val.upload(value_vectors);
    d_tie.upload(encode_tiebreak);
    uint32_t* enc = fold->enc.ptr;
    uint64_t bad = ~0ull;
    // streamed staging (one persistent encoder launch per row set, fed by the
    // host copies; HVB200_STAGE_STREAM=0 selects the chunked pipeline)
    const char* se = getenv("HVB200_STAGE_STREAM");
    bool streamed = !(se && atoi(se) == 0);
    DevBuf<uint8_t> d_bins;
    DevBuf<unsigned long long> d_ready;
    if (streamed) {
      d_bins = DevBuf<uint8_t>(rows * ldb, st);
      d_ready = DevBuf<unsigned long long>(2, st);
      sync(ctx);
      bad = encode_host_bins_streamed(ctx, train_bins, train_rows, features, bins, dim, d_id.ptr, d_val.ptr,
                                      d_tie.ptr, d_bins.ptr, enc, ldw, ctx->stream, d_ready.ptr, streamed);
      if (streamed && bad == ~0ull) {
        // the train labels go up on the aux stream while the train rows encode
        // (a pageable upload is synchronous for the host, so it is issued after
        // the host has fed the launch); the classical counts of the train rows
        // follow their launch on the main stream, the test rows' launch runs on aux
        ck(cudaMemcpyAsync(d_y.ptr, train_labels, train_rows * sizeof(int32_t), cudaMemcpyHostToDevice, ctx->aux),
           "H2D labels");
        cudaEvent_t ev;
        ck(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "event");
        ck(cudaEventRecord(ev, ctx->aux), "event");
        ck(cudaStreamWaitEvent(ctx->stream, ev, 0), "wait");
        cudaEventDestroy(ev);
        class_counts_device(ctx, ctx->stream, enc, train_rows, W, d_y.ptr, class_count, fold->counts.ptr,
                            fold->class_rows.ptr, ldw);
        bool s2 = false;
        bad = encode_host_bins_streamed(ctx, test_bins, test_rows, features, bins, dim, d_id.ptr, d_val.ptr,
                                        d_tie.ptr, d_bins.ptr + train_rows * ldb, enc + train_rows * ldw, ldw,
                                        ctx->aux, d_ready.ptr + 1, s2);
        if (!s2) fail(HV_ERR_CUDA, "fold: streamed encoder refused the test rows");
        if (bad != ~0ull) bad += train_rows * features;
      }
    }
    if (!streamed) {
      d_y.upload(train_labels);
      const size_t chunk = stage_chunk_rows(rows, features);
      DevBuf<uint8_t> b8[2] = {DevBuf<uint8_t>(chunk * ldb, st), DevBuf<uint8_t>(chunk * ldb, st)};
      sync(ctx);
      size_t k = 0;
      bad = encode_host_bins(ctx, train_bins, train_rows, features, bins, dim, HV_BIND_ID_LEVEL, d_id.ptr, d_val.ptr,
                             d_tie.ptr, [&](size_t r0, size_t) { return enc + r0 * ldw; }, b8, chunk, k, {}, ldw);
      if (bad == ~0ull) {
        // classical counts of the train rows overlap the staging/encode of the test rows
        cudaEvent_t ev;
        ck(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "event");
        ck(cudaEventRecord(ev, ctx->aux), "event");
        ck(cudaStreamWaitEvent(ctx->stream, ev, 0), "wait");
        cudaEventDestroy(ev);
        class_counts_device(ctx, ctx->stream, enc, train_rows, W, d_y.ptr, class_count, fold->counts.ptr,
                            fold->class_rows.ptr, ldw);
        bad = encode_host_bins(ctx, test_bins, test_rows, features, bins, dim, HV_BIND_ID_LEVEL, d_id.ptr, d_val.ptr,
                               d_tie.ptr, [&](size_t r0, size_t) { return enc + (train_rows + r0) * ldw; }, b8,
                               chunk, k, {}, ldw);
        if (bad != ~0ull) bad += train_rows * features;
      }
    }
    ck(cudaStreamSynchronize(ctx->aux), "sync aux");
    sync(ctx);
    unsigned long long l[kErrKinds];
    read_latch(ctx, l);
    if (l[kErrLabel] != ~0ull) reset_latch(ctx);
    // reference order (experiment.cpp:159-177): encode train, encode test, then train_classical
    if (bad != ~0ull) {
      const uint32_t b = bad < train_rows * features ? train_bins[bad] : test_bins[bad - train_rows * features];
      invalid("encode: feature " + std::to_string(bad % features) + " bin index " + std::to_string(b) +
              " out of range (bins = " + std::to_string(bins) + ")");
    }
    if (l[kErrLabel] != ~0ull) {
      invalid("train_classical: label " + std::to_string(train_labels[l[kErrLabel]]) + " at row " +
              std::to_string(l[kErrLabel]) + " out of range (classes = " + std::to_string(class_count) + ")");
    }
    *out = fold.release();
  });
}

hv_status hv_fold_counts(hv_fold* fold, void** counts_dev, void** class_rows_dev) {
  return guarded([&] {
    if (!fold) invalid("fold: null");
    if (counts_dev) *counts_dev = fold->counts.ptr;
    if (class_rows_dev) *class_rows_dev = fold->class_rows.ptr;
  });
}

hv_status hv_fold_predict(hv_context* ctx, hv_fold* fold, const uint32_t* model_tiebreak, int32_t* labels_out) {
  return guarded([&] {
    require(ctx);
    if (!fold) invalid("fold: null");
    cudaStream_t st = ctx->stream;
    DevBuf<uint32_t> tie(fold->W, st), cv(fold->C * fold->W, st);
    DevBuf<int32_t> lab(fold->test_rows, st);
    tie.upload(model_tiebreak);
    binarize_counts_device(ctx, st, fold->counts.ptr, fold->class_rows.ptr, fold->C, fold->D, tie.ptr, cv.ptr);
    const uint32_t* test = fold->enc.ptr + fold->train_rows * fold->ldw;
    DevBuf<uint32_t> packed;
    size_t ldq = fold->ldw;
    if (fold->C >= 32 && fold->ldw != fold->W) {  // the many-class scans read unpitched rows
      packed = DevBuf<uint32_t>(fold->test_rows * fold->W, st);
      ck(cudaMemcpy2DAsync(packed.ptr, fold->W * 4, test, fold->ldw * 4, fold->W * 4, fold->test_rows,
                           cudaMemcpyDeviceToDevice, st),
         "unpitch test rows");
      test = packed.ptr;
      ldq = fold->W;
    }
    predict_hamming_device(ctx, st, cv.ptr, fold->C, fold->D, test, fold->test_rows, lab.ptr, nullptr, nullptr, ldq);
    lab.download(labels_out);
    sync(ctx);
  });
}

void hv_fold_destroy(hv_fold* fold) { delete fold; }

// ---- dataset-resident folds (run_fold_packed, experiment.cpp:148-178) ----
hv_status hv_dataset_create(hv_context* ctx, const double* X, size_t rows, size_t features, const int32_t* labels,
                            hv_dataset** out) {
  return guarded([&] {
    require(ctx);
    if (!out) invalid("dataset: null output");
    *out = nullptr;
    if (rows == 0 || features == 0) invalid("dataset: empty matrix");
    auto ds = std::make_unique<hv_dataset>();
    ds->rows = rows;
    ds->F = features;
    ds->X = DevBuf<double>(rows * features, ctx->stream);
    ds->y = DevBuf<int32_t>(rows, ctx->stream);
    upload_host(ctx, X, rows * features * sizeof(double), ds->X.ptr);
    upload_host(ctx, labels, rows * sizeof(int32_t), ds->y.ptr);
    sync(ctx);
    *out = ds.release();
  });
}

void hv_dataset_destroy(hv_dataset* ds) { delete ds; }

}  // extern "C"

namespace hvb {
namespace {
// run_fold_packed (experiment.cpp:148-178) on a resident dataset; the test
// labels go to the host (labels_out) and/or are scattered on device into
// predicted[test row] (run_experiment's concatenation, experiment.cpp:305-310).
void dataset_fold_impl(hv_context* ctx, const hv_dataset* ds, const uint64_t* train_idx, size_t n_train,
                       const uint64_t* test_idx, size_t n_test, size_t bins, const uint32_t* id_vectors,
                       const uint32_t* value_vectors, size_t dim, hv_binding binding, const uint32_t* encode_tiebreak,
                       size_t class_count, hv_metric metric, double gamma, const uint32_t* model_tiebreak, int online,
                       size_t batch_size, int32_t* labels_out, int32_t* predicted_dev, double* min_out,
                       double* max_out) {
  {
    if (!ds) invalid("dataset_fold: null dataset");
    // reference order: fit_discretizer, discretize, encode, train, predict
    if (n_train == 0) invalid("fit_discretizer: empty training matrix");
    if (bins < 2) invalid("fit_discretizer: need at least 2 bins");
    if (class_count == 0 || dim == 0) invalid("dataset_fold: classes and dim must be >= 1");
    if (online && batch_size == 0) invalid("train_online: batch_size must be >= 1");
    if (metric != HV_METRIC_HAMMING && metric != HV_METRIC_COSINE) fail(HV_ERR_LOGIC, "bad Metric");
    check_indices(train_idx, n_train, ds->rows, "train");
    check_indices(test_idx, n_test, ds->rows, "test");
    cudaStream_t st = ctx->stream;
    const size_t F = ds->F, C = class_count, D = dim, W = words_per_row(D), ldb = bins_pitch(F);
    const size_t n = n_train + n_test;
    DevBuf<uint64_t> idx(n, st);
    ck(cudaMemcpyAsync(idx.ptr, train_idx, n_train * sizeof(uint64_t), cudaMemcpyHostToDevice, st), "H2D idx");
    if (n_test) {
      ck(cudaMemcpyAsync(idx.ptr + n_train, test_idx, n_test * sizeof(uint64_t), cudaMemcpyHostToDevice, st), "H2D idx");
    }
    DevBuf<double> mn(F, st), mx(F, st);
    fit_discretizer_device(ctx, st, ds->X.ptr, F, idx.ptr, n_train, mn.ptr, mx.ptr);
    DevBuf<uint8_t> b8(n * ldb, st);
    discretize_rows_device(ctx, st, ds->X.ptr, F, idx.ptr, n, mn.ptr, mx.ptr, bins, b8.ptr, ldb);
    DevBuf<uint32_t> d_id(F * W, st), d_val(bins * W, st), d_etb(W, st), d_mtb(W, st);
    d_id.upload(id_vectors);
    d_val.upload(value_vectors);
    d_etb.upload(encode_tiebreak);
    d_mtb.upload(model_tiebreak);
    // classical Hamming folds with < 32 classes keep the engine's pitched rows
    // (TMA-staged counts, uint4 / two-class predict); the online trainer and the
    // cosine scan read unpitched rows
    const bool pitched = !online && metric == HV_METRIC_HAMMING && C < 32;
    const size_t ldw = pitched ? hv_row_pitch_words(D) : W;
    DevBuf<uint32_t> enc(n * ldw, st);
    if (pitched && ldw != W) {
      encode_device(ctx, st, b8.ptr, ldb, n, F, d_id.ptr, d_val.ptr, bins, D, binding, d_etb.ptr, enc.ptr, true, 0, W,
                    ldw);
    } else {
      encode_device(ctx, st, b8.ptr, ldb, n, F, d_id.ptr, d_val.ptr, bins, D, binding, d_etb.ptr, enc.ptr);
    }
    DevBuf<int32_t> ytr(n_train, st), lab(std::max<size_t>(n_test, 1), st);
    gather_labels_kernel<<<sgrid(ctx, n_train, 256), 256, 0, st>>>(ds->y.ptr, idx.ptr, n_train, ytr.ptr);
    launched("gather_labels_kernel");
    DevBuf<double> acc(C * D, st), weight(C, st);
    DevBuf<uint64_t> counts(C, st);
    DevBuf<uint32_t> cv(C * W, st);
    if (online) {
      // labels are validated by the bootstrap's classical counts (first batch)
      // and, for later batches, below against the label latch
      check_labels_device(ctx, st, ytr.ptr, n_train, C);
      train_online_device(ctx, st, metric, enc.ptr, n_train, D, ytr.ptr, C, batch_size, gamma, d_mtb.ptr, acc.ptr,
                          weight.ptr, counts.ptr, cv.ptr);
    } else {
      DevBuf<uint32_t> cnt(C * 32 * W, st);
      cnt.zero();
      counts.zero();
      class_counts_device(ctx, st, enc.ptr, n_train, W, ytr.ptr, C, cnt.ptr, counts.ptr, ldw);
      binarize_counts_device(ctx, st, cnt.ptr, counts.ptr, C, D, d_mtb.ptr, cv.ptr);
      if (metric == HV_METRIC_COSINE) {
        init_from_counts_kernel<<<sgrid(ctx, C * D, 256), 256, 0, st>>>(cnt.ptr, counts.ptr, C, D, W, acc.ptr,
                                                                        weight.ptr, counts.ptr);
        launched("init_from_counts_kernel");
      }
    }
    if (n_test) {
      const uint32_t* q = enc.ptr + n_train * ldw;
      if (metric == HV_METRIC_HAMMING) {
        predict_hamming_device(ctx, st, cv.ptr, C, D, q, n_test, lab.ptr, nullptr, nullptr, ldw);
      } else {
        DevBuf<double> sc(n_test * C, st);
        cosine_scores_device(ctx, st, acc.ptr, C, D, q, n_test, sc.ptr, 0);
        argmax_kernel<<<sgrid(ctx, n_test, 128), 128, 0, st>>>(sc.ptr, n_test, static_cast<uint32_t>(C), lab.ptr);
        launched("argmax_kernel");
      }
      if (labels_out) {
        ck(cudaMemcpyAsync(labels_out, lab.ptr, n_test * sizeof(int32_t), cudaMemcpyDeviceToHost, st), "D2H labels");
      }
      if (predicted_dev) scatter_labels_device(ctx, st, idx.ptr + n_train, n_test, lab.ptr, predicted_dev);
    }
    if (min_out) mn.download(min_out);
    if (max_out) mx.download(max_out);
    sync(ctx);
    unsigned long long l[kErrKinds];
    read_latch(ctx, l);
    if (l[kErrLabel] != ~0ull || l[kErrZeroQuery] != ~0ull) {
      reset_latch(ctx);
      if (l[kErrLabel] != ~0ull) {
        int32_t bad = 0;
        const uint64_t k = l[kErrLabel];
        ck(cudaMemcpy(&bad, ytr.ptr + k, sizeof(int32_t), cudaMemcpyDeviceToHost), "D2H label");
        // model.cpp:282-301: the bootstrap batch is checked by train_classical,
        // every batch again by online_update (row index within the batch)
        const bool boot = !online || k < std::min(batch_size, n_train);
        const uint64_t row = boot ? k : k - (k / batch_size) * batch_size;
        invalid(std::string(boot ? "train_classical" : "online_update") + ": label " + std::to_string(bad) + " at row " +
                std::to_string(row) + " out of range (classes = " + std::to_string(C) + ")");
      }
      fail(HV_ERR_DOMAIN, "cosine_similarity: zero query vector");
    }
  }
}
}  // namespace
}  // namespace hvb

struct hv_experiment {
  const hv_dataset* ds = nullptr;
  hvb::DevBuf<int32_t> predicted;  // rows, -1 = untested
};

extern "C" {

hv_status hv_dataset_fold(hv_context* ctx, const hv_dataset* ds, const uint64_t* train_idx, size_t n_train,
                          const uint64_t* test_idx, size_t n_test, size_t bins, const uint32_t* id_vectors,
                          const uint32_t* value_vectors, size_t dim, hv_binding binding,
                          const uint32_t* encode_tiebreak, size_t class_count, hv_metric metric, double gamma,
                          const uint32_t* model_tiebreak, int online, size_t batch_size, int32_t* labels_out,
                          double* min_out, double* max_out) {
  return guarded([&] {
    require(ctx);
    if (n_test && !labels_out) invalid("dataset_fold: null labels_out");
    dataset_fold_impl(ctx, ds, train_idx, n_train, test_idx, n_test, bins, id_vectors, value_vectors, dim, binding,
                      encode_tiebreak, class_count, metric, gamma, model_tiebreak, online, batch_size, labels_out,
                      nullptr, min_out, max_out);
  });
}

hv_status hv_experiment_create(hv_context* ctx, const hv_dataset* ds, hv_experiment** out) {
  return guarded([&] {
    require(ctx);
    if (!ds || !out) invalid("experiment_create: null dataset or output");
    auto ex = std::make_unique<hv_experiment>();
    ex->ds = ds;
    ex->predicted = DevBuf<int32_t>(std::max<size_t>(ds->rows, 1), ctx->stream);
    ck(cudaMemsetAsync(ex->predicted.ptr, 0xFF, ex->predicted.bytes(), ctx->stream), "memset");
    sync(ctx);
    *out = ex.release();
  });
}

void hv_experiment_destroy(hv_experiment* ex) { delete ex; }

hv_status hv_experiment_fold(hv_context* ctx, hv_experiment* ex, const uint64_t* train_idx, size_t n_train,
                             const uint64_t* test_idx, size_t n_test, size_t bins, const uint32_t* id_vectors,
                             const uint32_t* value_vectors, size_t dim, hv_binding binding,
                             const uint32_t* encode_tiebreak, size_t class_count, hv_metric metric, double gamma,
                             const uint32_t* model_tiebreak, int online, size_t batch_size) {
  return guarded([&] {
    require(ctx);
    if (!ex) invalid("experiment_fold: null experiment");
    dataset_fold_impl(ctx, ex->ds, train_idx, n_train, test_idx, n_test, bins, id_vectors, value_vectors, dim,
                      binding, encode_tiebreak, class_count, metric, gamma, model_tiebreak, online, batch_size,
                      nullptr, ex->predicted.ptr, nullptr, nullptr);
  });
}

hv_status hv_experiment_finish(hv_context* ctx, hv_experiment* ex, size_t class_count, size_t smooth_window,
                               int positive_class, hv_eval_report* report, uint64_t* n_tested,
                               uint64_t* tested_rows, int32_t* truth, int32_t* predicted, int32_t* final_labels) {
  return guarded([&] {
    require(ctx);
    if (!ex) invalid("experiment_finish: null experiment");
    cudaStream_t st = ctx->stream;
    DevBuf<uint64_t> tested;
    DevBuf<int32_t> pred_seq, truth_seq;
    const size_t m = compact_tested_device(ctx, st, ex->predicted.ptr, ex->ds->y.ptr, ex->ds->rows, tested, pred_seq,
                                           truth_seq);
    if (m == 0) invalid("no test samples produced by split");
    // experiment.cpp:331-336: smoothing only for binary runs
    const bool smooth = class_count == 2 && smooth_window > 1;
    DevBuf<int32_t> fin;
    const int32_t* final_seq = pred_seq.ptr;
    if (smooth) {
      fin = DevBuf<int32_t>(m, st);
      smooth_labels_device(ctx, st, pred_seq.ptr, m, smooth_window, fin.ptr);
      final_seq = fin.ptr;
    }
    DevBuf<unsigned long long> counts(8, st);
    confusion_device(ctx, st, final_seq, truth_seq.ptr, m, positive_class, counts.ptr);
    episodes_device(ctx, st, final_seq, truth_seq.ptr, m, positive_class, counts.ptr + 5);
    unsigned long long h[8];
    counts.download(h);
    if (tested_rows) ck(cudaMemcpyAsync(tested_rows, tested.ptr, m * 8, cudaMemcpyDeviceToHost, st), "D2H");
    if (truth) ck(cudaMemcpyAsync(truth, truth_seq.ptr, m * 4, cudaMemcpyDeviceToHost, st), "D2H");
    if (predicted) ck(cudaMemcpyAsync(predicted, pred_seq.ptr, m * 4, cudaMemcpyDeviceToHost, st), "D2H");
    if (final_labels) ck(cudaMemcpyAsync(final_labels, final_seq, m * 4, cudaMemcpyDeviceToHost, st), "D2H");
    sync(ctx);
    if (report) fill_report(h, h + 5, m, report);
    if (n_tested) *n_tested = m;
  });
}

}  // extern "C"
