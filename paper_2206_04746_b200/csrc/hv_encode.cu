// hv_encode.cu — discretizer, bin narrowing, synthetic workload and the
// encoders (reference encoding.cpp:93-311).
//
// Encoding is the hot kernel of the whole pipeline. For ID-level binding
// (encoding.cpp:266-272, Eq. 1 of the paper) every output bit is the
// majority over F features of ID_f[j] ^ V_{bin_f}[j]. Instead of
// materialising the F x D bound matrix and transposing it (the reference's
// transpose-based vertical_sum, kernels.cpp:111-140), each thread owns one
// 32-bit output word and counts the 32 bit positions in parallel with a
// bit-sliced Harley–Seal carry-save network: ~2 LOP3 per bound word plus the
// XOR bind. The kernel is therefore integer-pipe bound, not HBM bound
// (SURVEY.md §8d): HBM traffic is F bytes of bins in and D/8 bytes out per
// datapoint.
//
// Two ID-level kernels:
//   - encode_tt_kernel (fast path): per-CTA shared-memory table
//     T[f][b] = ID_f ^ V_b for a slice of output words, one datapoint per
//     lane, bins staged through shared memory; the XOR bind disappears and
//     each bound word costs one conflict-free LDS + ~2 LOP3.
//   - encode_generic_kernel: one thread per (row, word), codebook words read
//     through L1/L2; handles every binding/shape the fast path does not.

#include <algorithm>
#include <vector>

#include "hv_internal.cuh"
#include "hv_stage.h"
#include "hvb200_synth.h"

namespace hvb {

// ------------------------------------------------------------ narrow ----
// uint32 bins (rows x F) -> uint8 bins with row pitch ldb (zero padded),
// validating bin < B (encoding.cpp:43-55). One thread per 4 output bytes.
__global__ void narrow_bins_kernel(const uint32_t* __restrict__ in, uint64_t rows, uint32_t F, uint32_t B,
                                   uint8_t* __restrict__ out, uint32_t ldb, uint64_t flat_base,
                                   unsigned long long* err) {
  const uint32_t quads = ldb >> 2;
  const uint64_t total = rows * quads;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t r = i / quads;
    const uint32_t f0 = static_cast<uint32_t>(i % quads) * 4u;
    uint32_t packed = 0;
#pragma unroll
    for (uint32_t t = 0; t < 4; ++t) {
      const uint32_t f = f0 + t;
      if (f < F) {
        const uint32_t b = in[r * F + f];
        if (b >= B) latch(err, kErrBin, flat_base + r * F + f);
        packed |= (b < B ? b : 0u) << (8u * t);
      }
    }
    reinterpret_cast<uint32_t*>(out + r * ldb)[f0 >> 2] = packed;
  }
}

// ------------------------------------------------------- discretizer ----
// encoding.cpp:93-119. Ordered two-level reduction so that the strict
// first-row-initialised semantics (including NaN in row 0 and signed zeros)
// are reproduced exactly: partials over rows >= 1 start at +/-inf and only
// move on strict </>, then partials are folded into row 0 in row order.
__global__ void minmax_partial_kernel(const double* __restrict__ data, uint64_t rows, uint32_t F,
                                      uint64_t rows_per_block, double* __restrict__ pmin,
                                      double* __restrict__ pmax, const uint64_t* __restrict__ idx = nullptr) {
  const uint32_t f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= F) return;
  const uint64_t r0 = 1 + blockIdx.y * rows_per_block;
  const uint64_t r1 = min(rows, r0 + rows_per_block);
  double mn = __longlong_as_double(0x7FF0000000000000ll);   // +inf
  double mx = __longlong_as_double(0xFFF0000000000000ull);  // -inf
  for (uint64_t r = r0; r < r1; ++r) {
    const double v = data[(idx ? idx[r] : r) * F + f];
    if (v < mn) mn = v;
    if (v > mx) mx = v;
  }
  pmin[static_cast<uint64_t>(blockIdx.y) * F + f] = mn;
  pmax[static_cast<uint64_t>(blockIdx.y) * F + f] = mx;
}

__global__ void minmax_final_kernel(const double* __restrict__ data, uint32_t F, uint32_t nblocks,
                                    const double* __restrict__ pmin, const double* __restrict__ pmax,
                                    double* __restrict__ mn_out, double* __restrict__ mx_out,
                                    const uint64_t* __restrict__ idx = nullptr) {
  const uint32_t f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= F) return;
  const uint64_t r0 = idx ? idx[0] : 0;
  double mn = data[r0 * F + f], mx = data[r0 * F + f];
  for (uint32_t b = 0; b < nblocks; ++b) {
    const double a = pmin[static_cast<uint64_t>(b) * F + f];
    const double c = pmax[static_cast<uint64_t>(b) * F + f];
    if (a < mn) mn = a;
    if (c > mx) mx = c;
  }
  mn_out[f] = mn;
  mx_out[f] = mx;
}

// encoding.cpp:121-139: bin = floor((x - min) / (max - min) * B), clamped;
// degenerate features and NaN map to 0. Explicit _rn intrinsics keep the
// arithmetic identical to the host's IEEE evaluation (no contraction).
template <class OutT>
__global__ void discretize_kernel(const double* __restrict__ data, uint64_t rows, uint32_t F,
                                  const double* __restrict__ mn, const double* __restrict__ mx, uint32_t B,
                                  OutT* __restrict__ out, uint32_t ld_out, const uint64_t* __restrict__ idx = nullptr) {
  const uint64_t total = rows * F;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t r = i / F;
    const uint32_t f = static_cast<uint32_t>(i % F);
    const double lo = mn[f], hi = mx[f];
    const double x = data[(idx ? idx[r] : r) * F + f];
    uint32_t b = 0;
    if (!(lo == hi)) {
      const double t = floor(__dmul_rn(__ddiv_rn(__dsub_rn(x, lo), __dsub_rn(hi, lo)), static_cast<double>(B)));
      const double top = static_cast<double>(B - 1);
      if (t >= top) b = B - 1;
      else if (t > 0.0) b = static_cast<uint32_t>(t);
    }
    out[r * ld_out + f] = static_cast<OutT>(b);
  }
}

// ------------------------------------------------------------- synth ----
__global__ void synth_kernel(uint64_t row0, uint64_t rows, uint32_t F, uint32_t C, uint32_t B, int kind,
                             uint64_t seed, uint8_t* __restrict__ bins8, uint32_t ldb, int32_t* __restrict__ labels) {
  const uint64_t total = rows * ldb;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t r = i / ldb;
    const uint32_t f = static_cast<uint32_t>(i % ldb);
    const int32_t y = hvs_label(row0 + r, C, kind);
    bins8[i] = f < F ? static_cast<uint8_t>(hvs_bin(row0 + r, f, F, y, B, seed)) : 0;
    if (f == 0 && labels) labels[r] = y;
  }
}

// ----------------------------------------------------- generic encode ----
// One thread per (row, output word); features consumed 16 at a time by the
// Harley–Seal counter. PERM: bound word = rotate(V_b, f) (encoding.cpp:273-279).
template <int NH, bool PERM>
__global__ void __launch_bounds__(256) encode_generic_kernel(const uint8_t* __restrict__ bins8, uint32_t ldb,
                                                             uint64_t rows, uint32_t F,
                                                             const uint32_t* __restrict__ id,
                                                             const uint32_t* __restrict__ val, uint32_t D,
                                                             uint32_t W, const uint32_t* __restrict__ tie,
                                                             uint32_t* __restrict__ out) {
  const uint64_t total = rows * W;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t r = i / W;
    const uint32_t w = static_cast<uint32_t>(i % W);
    const uint8_t* b = bins8 + r * ldb;
    HSCounter<NH> h;
    for (uint32_t f0 = 0; f0 < F; f0 += 16) {
      uint32_t x[16];
#pragma unroll
      for (int t = 0; t < 16; ++t) {
        const uint32_t f = f0 + t;
        uint32_t v = 0;
        if (f < F) {
          const uint32_t* vrow = val + static_cast<uint64_t>(b[f]) * W;
          if (PERM) {
            const uint32_t p = static_cast<uint32_t>((static_cast<uint64_t>(w) * 32u + D - (f % D)) % D);
            v = get_bits_cyclic(vrow, W, D, p);
          } else {
            v = id[static_cast<uint64_t>(f) * W + w] ^ vrow[w];
          }
        }
        x[t] = v;
      }
      h.add16(x);
    }
    out[i] = h.majority(F, tie[w]) & valid_mask(w, D);
  }
}

// encoding.cpp:280-290: appending concatenates the first floor(D/F) bits of
// each V_{bin_f}; the remainder bits stay zero. One thread per output word.
__global__ void encode_append_kernel(const uint8_t* __restrict__ bins8, uint32_t ldb, uint64_t rows, uint32_t F,
                                     const uint32_t* __restrict__ val, uint32_t D, uint32_t W, uint32_t seg,
                                     uint32_t* __restrict__ out) {
  const uint64_t total = rows * W;
  const uint64_t used = static_cast<uint64_t>(F) * seg;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t r = i / W;
    const uint32_t w = static_cast<uint32_t>(i % W);
    const uint8_t* b = bins8 + r * ldb;
    const uint64_t j0 = static_cast<uint64_t>(w) * 32u;
    const uint64_t j1 = min(j0 + 32u, used);
    uint32_t word = 0;
    for (uint64_t j = j0; j < j1;) {
      const uint32_t f = static_cast<uint32_t>(j / seg);
      const uint32_t off = static_cast<uint32_t>(j - static_cast<uint64_t>(f) * seg);
      const uint32_t len = static_cast<uint32_t>(min(j1 - j, static_cast<uint64_t>(seg - off)));
      uint32_t bits = get_bits32(val + static_cast<uint64_t>(b[f]) * W, W, off);
      if (len < 32u) bits &= (1u << len) - 1u;
      word |= bits << static_cast<uint32_t>(j - j0);
      j += len;
    }
    out[i] = word;
  }
}


}  // namespace hvb

using namespace hvb;

namespace hvb {

// Dispatch helpers -----------------------------------------------------------
template <bool PERM>
void launch_generic(hv_context* ctx, cudaStream_t st, int nh, const uint8_t* bins8, uint32_t ldb, uint64_t rows,
                    uint32_t F, const uint32_t* id, const uint32_t* val, uint32_t D, uint32_t W, const uint32_t* tie,
                    uint32_t* out) {
  const uint64_t items = rows * W;
  const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((items + 255) / 256, uint64_t(ctx->sm_count) * 16));
#define HV_GEN_CASE(N)                                                                                        \
  case N:                                                                                                     \
    encode_generic_kernel<N, PERM><<<grid, 256, 0, st>>>(bins8, ldb, rows, F, id, val, D, W, tie, out);       \
    break;
  switch (nh) {
    HV_GEN_CASE(1) HV_GEN_CASE(2) HV_GEN_CASE(3) HV_GEN_CASE(4) HV_GEN_CASE(5) HV_GEN_CASE(6)
    HV_GEN_CASE(7) HV_GEN_CASE(8) HV_GEN_CASE(9) HV_GEN_CASE(10) HV_GEN_CASE(11) HV_GEN_CASE(12)
    default: invalid("encode: feature count too large for the device encoder");
  }
#undef HV_GEN_CASE
  launched("encode_generic_kernel");
}

// Device-resident discretizer over an optional row-index subset (datasets kept
// in HBM across folds): fit = the ordered first-row min/max of encoding.cpp:
// 93-119 over rows idx[0..n); discretize writes uint8 bins with pitch ldb.
void fit_discretizer_device(hv_context* ctx, cudaStream_t st, const double* X, size_t F, const uint64_t* idx,
                            size_t n, double* mn, double* mx) {
  const uint64_t rpb = 4096;
  const uint32_t nblocks = static_cast<uint32_t>(n > 1 ? (n - 1 + rpb - 1) / rpb : 0);
  DevBuf<double> pmin(std::max<size_t>(1, nblocks) * F, st), pmax(std::max<size_t>(1, nblocks) * F, st);
  if (nblocks) {
    dim3 grid(grid_for(F, 128), nblocks);
    minmax_partial_kernel<<<grid, 128, 0, st>>>(X, n, static_cast<uint32_t>(F), rpb, pmin.ptr, pmax.ptr, idx);
    launched("minmax_partial_kernel");
  }
  minmax_final_kernel<<<grid_for(F, 128), 128, 0, st>>>(X, static_cast<uint32_t>(F), nblocks, pmin.ptr, pmax.ptr, mn,
                                                         mx, idx);
  launched("minmax_final_kernel");
}

void discretize_rows_device(hv_context* ctx, cudaStream_t st, const double* X, size_t F, const uint64_t* idx,
                            size_t n, const double* mn, const double* mx, size_t B, uint8_t* out, size_t ldb) {
  check_bins_u8(B, "discretize");
  if (n == 0) return;
  ck(cudaMemsetAsync(out, 0, n * ldb, st), "memset bins");
  const uint64_t items = n * F;
  const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((items + 255) / 256, uint64_t(ctx->sm_count) * 16));
  discretize_kernel<uint8_t><<<grid, 256, 0, st>>>(X, n, static_cast<uint32_t>(F), mn, mx, static_cast<uint32_t>(B),
                                                   out, static_cast<uint32_t>(ldb), idx);
  launched("discretize_kernel");
}

// Encodes validated uint8 bins on stream `st`.
void encode_device(hv_context* ctx, cudaStream_t st, const uint8_t* bins8, size_t ldb, size_t rows, size_t F,
                   const uint32_t* id, const uint32_t* val, size_t B, size_t D, hv_binding binding,
                   const uint32_t* tie, uint32_t* out, bool allow_fast, size_t w0, size_t wcount, size_t ldo) {
  check_bins_u8(B, "encode");
  const size_t W = words_per_row(D);
  if (rows == 0 || W == 0) return;
  if (D > 0xFFFFFFFFull || F > 0xFFFFFFFFull) invalid("encode: shape too large");
  if (wcount == 0) {
    w0 = 0;
    wcount = W;
    ldo = W;
  }
  if (w0 + wcount > W || ldo < wcount) invalid("encode: word range outside the row");
  // the tensor-core encoder (HVB200_ENCODE_TC=1 while it is being evaluated)
  if (binding == HV_BIND_ID_LEVEL && allow_fast && w0 == 0 && wcount == W) {
    const char* tc = getenv("HVB200_ENCODE_TC");
    if (tc && tc[0] == '1' &&
        launch_tc(ctx, st, bins8, static_cast<uint32_t>(ldb), rows, static_cast<uint32_t>(F), id, val,
                  static_cast<uint32_t>(B), static_cast<uint32_t>(D), static_cast<uint32_t>(W), tie, out,
                  static_cast<uint32_t>(ldo))) {
      return;
    }
  }
  if (wcount != W || ldo != W) {
    // a column slice: the fused encoder writes it directly; other bindings
    // encode whole rows into scratch and copy the slice out
    if ((binding == HV_BIND_ID_LEVEL || binding == HV_BIND_PERMUTATION) && allow_fast &&
        launch_tt(ctx, st, bins8, static_cast<uint32_t>(ldb), rows, static_cast<uint32_t>(F), id, val,
                  static_cast<uint32_t>(B), static_cast<uint32_t>(D), static_cast<uint32_t>(W), tie, out,
                  static_cast<uint32_t>(w0), static_cast<uint32_t>(wcount), static_cast<uint32_t>(ldo),
                  binding == HV_BIND_PERMUTATION)) {
      return;
    }
    DevBuf<uint32_t> full(rows * W, st);
    encode_device(ctx, st, bins8, ldb, rows, F, id, val, B, D, binding, tie, full.ptr, allow_fast);
    ck(cudaMemcpy2DAsync(out, ldo * 4, full.ptr + w0, W * 4, wcount * 4, rows, cudaMemcpyDeviceToDevice, st),
       "slice copy");
    return;
  }
  switch (binding) {
    case HV_BIND_ID_LEVEL:
      if (allow_fast && launch_tt(ctx, st, bins8, static_cast<uint32_t>(ldb), rows, static_cast<uint32_t>(F), id, val,
                                  static_cast<uint32_t>(B), static_cast<uint32_t>(D), static_cast<uint32_t>(W), tie, out,
                                  0u, static_cast<uint32_t>(W), static_cast<uint32_t>(W))) {
        return;
      }
      launch_generic<false>(ctx, st, hs_high_planes(F), bins8, static_cast<uint32_t>(ldb), rows,
                            static_cast<uint32_t>(F), id, val, static_cast<uint32_t>(D), static_cast<uint32_t>(W), tie,
                            out);
      return;
    case HV_BIND_PERMUTATION:
      // the table encoder with rotated level vectors as its bound words
      if (allow_fast && launch_tt(ctx, st, bins8, static_cast<uint32_t>(ldb), rows, static_cast<uint32_t>(F), id, val,
                                  static_cast<uint32_t>(B), static_cast<uint32_t>(D), static_cast<uint32_t>(W), tie, out,
                                  0u, static_cast<uint32_t>(W), static_cast<uint32_t>(W), true)) {
        return;
      }
      launch_generic<true>(ctx, st, hs_high_planes(F), bins8, static_cast<uint32_t>(ldb), rows,
                           static_cast<uint32_t>(F), id, val, static_cast<uint32_t>(D), static_cast<uint32_t>(W), tie,
                           out);
      return;
    case HV_BIND_APPENDING: {
      const size_t seg = D / F;
      if (seg == 0) invalid("encode: appending needs dim >= feature count");
      const uint64_t items = rows * W;
      const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((items + 255) / 256, uint64_t(ctx->sm_count) * 16));
      encode_append_kernel<<<grid, 256, 0, st>>>(bins8, static_cast<uint32_t>(ldb), rows, static_cast<uint32_t>(F), val,
                                                 static_cast<uint32_t>(D), static_cast<uint32_t>(W),
                                                 static_cast<uint32_t>(seg), out);
      launched("encode_append_kernel");
      return;
    }
  }
  fail(HV_ERR_LOGIC, "bad BindingStrategy");
}

void narrow_device(hv_context* ctx, cudaStream_t st, const uint32_t* bins32, size_t rows, size_t F, size_t B,
                   uint8_t* bins8, size_t ldb, uint64_t flat_base) {
  check_bins_u8(B, "narrow_bins");
  if (rows == 0) return;
  const uint64_t items = rows * (ldb / 4);
  const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((items + 255) / 256, uint64_t(ctx->sm_count) * 16));
  narrow_bins_kernel<<<grid, 256, 0, st>>>(bins32, rows, static_cast<uint32_t>(F), static_cast<uint32_t>(B), bins8,
                                          static_cast<uint32_t>(ldb), flat_base, ctx->d_err);
  launched("narrow_bins_kernel");
}

}  // namespace hvb

extern "C" {

hv_status hv_fit_discretizer(hv_context* ctx, const double* data, size_t rows, size_t features, size_t bins,
                             double* min_out, double* max_out) {
  return guarded([&] {
    require(ctx);
    if (rows == 0 || features == 0) invalid("fit_discretizer: empty training matrix");
    if (bins < 2) invalid("fit_discretizer: need at least 2 bins");
    const uint64_t rpb = 4096;
    const uint32_t nblocks = static_cast<uint32_t>(rows > 1 ? (rows - 1 + rpb - 1) / rpb : 0);
    DevBuf<double> d(rows * features, ctx->stream), pmin(std::max<size_t>(1, nblocks) * features, ctx->stream),
        pmax(std::max<size_t>(1, nblocks) * features, ctx->stream), omin(features, ctx->stream),
        omax(features, ctx->stream);
    d.upload(data);
    if (nblocks) {
      dim3 grid(grid_for(features, 128), nblocks);
      minmax_partial_kernel<<<grid, 128, 0, ctx->stream>>>(d.ptr, rows, static_cast<uint32_t>(features), rpb, pmin.ptr,
                                                           pmax.ptr);
      launched("minmax_partial_kernel");
    }
    minmax_final_kernel<<<grid_for(features, 128), 128, 0, ctx->stream>>>(d.ptr, static_cast<uint32_t>(features),
                                                                           nblocks, pmin.ptr, pmax.ptr, omin.ptr,
                                                                           omax.ptr);
    launched("minmax_final_kernel");
    omin.download(min_out);
    omax.download(max_out);
    sync(ctx);
  });
}

hv_status hv_discretize_matrix(hv_context* ctx, const double* data, size_t rows, size_t features, const double* mn,
                               const double* mx, size_t bins, uint32_t* out) {
  return guarded([&] {
    require(ctx);
    if (rows * features == 0) return;
    DevBuf<double> d(rows * features, ctx->stream), dmn(features, ctx->stream), dmx(features, ctx->stream);
    DevBuf<uint32_t> o(rows * features, ctx->stream);
    d.upload(data);
    dmn.upload(mn);
    dmx.upload(mx);
    const uint64_t items = rows * features;
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((items + 255) / 256, uint64_t(ctx->sm_count) * 16));
    discretize_kernel<uint32_t><<<grid, 256, 0, ctx->stream>>>(d.ptr, rows, static_cast<uint32_t>(features), dmn.ptr,
                                                              dmx.ptr, static_cast<uint32_t>(bins), o.ptr,
                                                              static_cast<uint32_t>(features));
    launched("discretize_kernel");
    o.download(out);
    sync(ctx);
  });
}

hv_status hv_encode_batch(hv_context* ctx, const uint32_t* bin_rows, size_t rows, size_t features,
                          const uint32_t* id_vectors, const uint32_t* value_vectors, size_t bins, size_t dim,
                          hv_binding binding, const uint32_t* tiebreak, size_t tiebreak_rows, size_t tiebreak_dim,
                          uint32_t* out) {
  return guarded([&] {
    require(ctx);
    if (rows == 0) return;
    if (binding != HV_BIND_ID_LEVEL && binding != HV_BIND_PERMUTATION && binding != HV_BIND_APPENDING) {
      fail(HV_ERR_LOGIC, "bad BindingStrategy");
    }
    // encode() checks, in the reference's order, for the first row
    // (encoding.cpp:43-55, 262-264, 283), then every row's bins on device.
    for (size_t f = 0; f < features; ++f) {
      if (bin_rows[f] >= bins) {
        invalid("encode: feature " + std::to_string(f) + " bin index " + std::to_string(bin_rows[f]) +
                " out of range (bins = " + std::to_string(bins) + ")");
      }
    }
    if (tiebreak_rows != 1 || tiebreak_dim != dim) invalid("encode: tiebreak must be 1 x dim");
    if (binding == HV_BIND_APPENDING && (features == 0 || dim / features == 0)) {
      invalid("encode: appending needs dim >= feature count");
    }
    if (features == 0 || dim == 0) invalid("encode: features and dim must be >= 1");
    const size_t W = words_per_row(dim);
    const size_t ldb = bins_pitch(features);
    DevBuf<uint32_t> d_id(features * W, ctx->stream), d_val(bins * W, ctx->stream), d_tie(W, ctx->stream);
    d_id.upload(id_vectors);
    d_val.upload(value_vectors);
    d_tie.upload(tiebreak);
    sync(ctx);
    // Host narrowing into pinned slots -> H2D -> encode -> D2H, chunked over
    // the context's two streams (hv_stage.cu).
    const size_t chunk = stage_chunk_rows(rows, features);
    DevBuf<uint8_t> b8[2] = {DevBuf<uint8_t>(chunk * ldb, ctx->stream), DevBuf<uint8_t>(chunk * ldb, ctx->stream)};
    DevBuf<uint32_t> o[2] = {DevBuf<uint32_t>(chunk * W, ctx->stream), DevBuf<uint32_t>(chunk * W, ctx->stream)};
    sync(ctx);
    size_t k = 0;
    const uint64_t bad = encode_host_bins(
        ctx, bin_rows, rows, features, bins, dim, binding, d_id.ptr, d_val.ptr, d_tie.ptr,
        [&](size_t, size_t kk) { return o[kk & 1].ptr; }, b8, chunk, k,
        [&](size_t r0, size_t n, size_t kk, cudaStream_t st) {
          ck(cudaMemcpyAsync(out + r0 * W, o[kk & 1].ptr, n * W * 4, cudaMemcpyDeviceToHost, st), "D2H encoded");
        });
    ck(cudaStreamSynchronize(ctx->aux), "sync aux");
    sync(ctx);
    if (bad != ~0ull) {
      invalid("encode: feature " + std::to_string(bad % features) + " bin index " + std::to_string(bin_rows[bad]) +
              " out of range (bins = " + std::to_string(bins) + ")");
    }
  });
}

hv_status hv_dev_narrow_bins(hv_context* ctx, const uint32_t* bins32, size_t rows, size_t features, size_t bins,
                             uint8_t* bins8, size_t ldb) {
  return guarded([&] {
    require(ctx);
    if (ldb < features || ldb % 4) invalid("narrow_bins: ldb must be >= features and a multiple of 4");
    narrow_device(ctx, ctx->stream, bins32, rows, features, bins, bins8, ldb, 0);
  });
}

hv_status hv_dev_encode(hv_context* ctx, const uint8_t* bins8, size_t ldb, size_t rows, size_t features,
                        const uint32_t* id_vectors, const uint32_t* value_vectors, size_t bins, size_t dim,
                        hv_binding binding, const uint32_t* tiebreak, uint32_t* out) {
  return guarded([&] {
    require(ctx);
    if (features == 0 || dim == 0) invalid("encode: features and dim must be >= 1");
    if (ldb < features) invalid("encode: ldb < features");
    const char* env = getenv("HVB200_ENCODE_GENERIC");
    encode_device(ctx, ctx->stream, bins8, ldb, rows, features, id_vectors, value_vectors, bins, dim, binding, tiebreak,
                  out, !(env && env[0] == '1'));
  });
}

hv_status hv_dev_encode_words(hv_context* ctx, const uint8_t* bins8, size_t ldb, size_t rows, size_t features,
                              const uint32_t* id_vectors, const uint32_t* value_vectors, size_t bins, size_t dim,
                              hv_binding binding, const uint32_t* tiebreak, size_t word_begin, size_t word_count,
                              uint32_t* out, size_t ldo) {
  return guarded([&] {
    require(ctx);
    if (features == 0 || dim == 0) invalid("encode: features and dim must be >= 1");
    if (ldb < features) invalid("encode: ldb < features");
    if (word_count == 0) invalid("encode_words: word_count must be >= 1");
    const char* env = getenv("HVB200_ENCODE_GENERIC");
    encode_device(ctx, ctx->stream, bins8, ldb, rows, features, id_vectors, value_vectors, bins, dim, binding, tiebreak,
                  out, !(env && env[0] == '1'), word_begin, word_count, ldo);
  });
}

hv_status hv_dev_synth(hv_context* ctx, uint64_t row0, size_t rows, size_t features, size_t class_count, size_t bins,
                       int label_kind, uint64_t seed, uint8_t* bins8, size_t ldb, int32_t* labels) {
  return guarded([&] {
    require(ctx);
    if (ldb < features) invalid("synth: ldb < features");
    if (rows == 0) return;
    const uint64_t items = rows * ldb;
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((items + 255) / 256, uint64_t(ctx->sm_count) * 32));
    synth_kernel<<<grid, 256, 0, ctx->stream>>>(row0, rows, static_cast<uint32_t>(features),
                                                static_cast<uint32_t>(class_count), static_cast<uint32_t>(bins),
                                                label_kind, seed, bins8, static_cast<uint32_t>(ldb), labels);
    launched("synth_kernel");
  });
}

}  // extern "C"
