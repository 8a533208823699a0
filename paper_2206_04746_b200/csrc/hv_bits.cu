// hv_bits.cu — packed bit-matrix kernels (reference kernels.hpp:16-63):
// pack / unpack / xor_bind / rotate / horizontal_sum / transpose /
// vertical_sum / majority_binarize, plus the shared column-count kernel that
// classical training also uses.
//
// All kernels are HBM-streaming integer work: coalesced 32-bit word access
// (a warp covers 128 contiguous bytes), grid-stride loops sized to the SM
// count, no shared-memory staging needed except where noted.

#include <vector>

#include "hv_internal.cuh"

namespace hvb {

// --------------------------------------------------------------- pack ----
// kernels.cpp:44-61. One thread per output word; validates bytes <= 1.
__global__ void pack_kernel(const uint8_t* __restrict__ dense, uint64_t rows, uint32_t dim, uint32_t W,
                            uint32_t* __restrict__ out, unsigned long long* err) {
  const uint64_t total = rows * W;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t r = i / W;
    const uint32_t w = static_cast<uint32_t>(i % W);
    const uint8_t* src = dense + r * dim + w * 32u;
    const uint32_t n = min(32u, dim - w * 32u);
    uint32_t word = 0;
    for (uint32_t t = 0; t < n; ++t) {
      const uint32_t b = src[t];
      if (b > 1u) latch(err, kErrByte, r * dim + w * 32u + t);
      word |= (b & 1u) << t;
    }
    out[i] = word;
  }
}

// kernels.cpp:63-73. One thread per input word, 32 byte stores.
__global__ void unpack_kernel(const uint32_t* __restrict__ words, uint64_t rows, uint32_t dim, uint32_t W,
                              uint8_t* __restrict__ dense) {
  const uint64_t total = rows * W;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t r = i / W;
    const uint32_t w = static_cast<uint32_t>(i % W);
    const uint32_t v = words[i];
    uint8_t* dst = dense + r * dim + w * 32u;
    const uint32_t n = min(32u, dim - w * 32u);
    for (uint32_t t = 0; t < n; ++t) dst[t] = static_cast<uint8_t>((v >> t) & 1u);
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
// perm[p] (or p) for p in [0, seg_off[nseg]). One thread per word column;
// blockIdx.y walks chunks of `chunk` positions (<= 2048 so 12-bit counters
// suffice); Harley–Seal accumulation, flushed with atomics at segment ends.
template <class CT>
__global__ void __launch_bounds__(128) column_count_kernel(const uint32_t* __restrict__ m, uint32_t W,
                                                           const uint32_t* __restrict__ perm,
                                                           const uint64_t* __restrict__ seg_off, uint32_t nseg,
                                                           uint64_t npos_fallback, uint32_t chunk, CT* single,
                                                           CT* const* __restrict__ dsts, uint32_t ndst) {
  const uint32_t w = blockIdx.x * blockDim.x + threadIdx.x;
  const bool active = w < W;
  const uint64_t npos = seg_off ? seg_off[nseg] : npos_fallback;
  uint64_t p0 = static_cast<uint64_t>(blockIdx.y) * chunk;
  if (p0 >= npos) return;
  const uint64_t p1 = min(npos, p0 + chunk);
  uint32_t s = 0;
  if (seg_off) {
    while (s + 1 < nseg && seg_off[s + 1] <= p0) ++s;
  }
  const uint64_t stride = 32ull * W;
  while (p0 < p1) {
    const uint64_t e = seg_off ? min(p1, seg_off[s + 1]) : p1;
    if (e > p0) {
      HSCounter<8> h;
      // 32 row loads in flight per thread; the permutation of the next batch
      // is fetched while this one's rows are loaded (two dependent loads per
      // batch would otherwise serialise)
      uint32_t rows_nx[32];
#pragma unroll
      for (int t = 0; t < 32; ++t) {
        const uint64_t q = p0 + t;
        rows_nx[t] = q < e ? (perm ? perm[q] : static_cast<uint32_t>(q)) : 0u;
      }
      for (uint64_t p = p0; p < e; p += 32) {
        uint32_t rr[32];
#pragma unroll
        for (int t = 0; t < 32; ++t) rr[t] = rows_nx[t];
        uint32_t x[32];
#pragma unroll
        for (int t = 0; t < 32; ++t) x[t] = (active && p + t < e) ? m[static_cast<uint64_t>(rr[t]) * W + w] : 0u;
        if (p + 32 < e) {
#pragma unroll
          for (int t = 0; t < 32; ++t) {
            const uint64_t q = p + 32 + t;
            rows_nx[t] = q < e ? (perm ? perm[q] : static_cast<uint32_t>(q)) : 0u;
          }
        }
        h.add16(x);
        h.add16(x + 16);
      }
      if (active) {
        // flush into every destination: the local counts, or — fused with the
        // all-reduce — the count buffers of all ranks over peer memory
        for (uint32_t d = 0; d < ndst; ++d) {
          CT* dst = (dsts ? dsts[d] : single) + s * stride + 32ull * w;
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

void launch_column_count_u32(cudaStream_t st, const uint32_t* m, uint32_t W, const uint32_t* perm,
                             const uint64_t* seg_off, uint32_t nseg, uint64_t max_pos, uint32_t* counts) {
  launch_column_count_peers(st, m, W, perm, seg_off, nseg, max_pos, counts, nullptr, 1);
}

void launch_column_count_peers(cudaStream_t st, const uint32_t* m, uint32_t W, const uint32_t* perm,
                               const uint64_t* seg_off, uint32_t nseg, uint64_t max_pos, uint32_t* single,
                               uint32_t* const* dsts_dev, uint32_t ndst) {
  if (max_pos == 0 || W == 0) return;
  if (max_pos > 0xFFFFFFFFull) invalid("class counts: more than 2^32 rows per call");
  const uint32_t chunk = 2048;
  dim3 grid(grid_for(W, 128), static_cast<unsigned>((max_pos + chunk - 1) / chunk));
  column_count_kernel<uint32_t><<<grid, 128, 0, st>>>(m, W, perm, seg_off, nseg, max_pos, chunk, single, dsts_dev,
                                                      dsts_dev ? ndst : 1u);
  launched("column_count_kernel");
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
    pack_kernel<<<stream_grid(ctx, rows * W, 256), 256, 0, ctx->stream>>>(d_in.ptr, rows, dim, W, d_out.ptr, ctx->d_err);
    launched("pack_kernel");
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
    unpack_kernel<<<stream_grid(ctx, rows * W, 256), 256, 0, ctx->stream>>>(d_in.ptr, rows, dim, W, d_out.ptr);
    launched("unpack_kernel");
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
    const uint32_t chunk = 2048;
    dim3 grid(grid_for(W, 128), static_cast<unsigned>((rows + chunk - 1) / chunk));
    if (rows > 0xFFFFFFFFull) invalid("vertical_sum: more than 2^32 rows");
    column_count_kernel<unsigned long long><<<grid, 128, 0, ctx->stream>>>(d_in.ptr, W, nullptr, nullptr, 1, rows,
                                                                          chunk, d_cnt.ptr, nullptr, 1);
    launched("column_count_kernel");
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
