// hv_encode_tt.cu — the fast ID-level encoder (reference encoding.cpp:266-272,
// the hot loop of the whole pipeline).
//
// Output bit j of datapoint i = majority over f < F of ID_f[j] ^ V_{bin(i,f)}[j].
// Per CTA, shared memory holds, for NC output words w_c,
//     T_c[f][b] = ID_f[w_c] ^ V_b[w_c]      (F16 x 16 words per table)
// so the XOR bind disappears: a bound word is one table lookup. Lane = datapoint,
// warp (c, g) = output word w_c for the 32 datapoints of group g. Per lane and
// bound word the cost is one conflict-free LDS (16 bins of one feature occupy
// 16 distinct banks; equal bins broadcast) plus a ~2.2-LOP3 share of a
// bit-sliced Harley–Seal carry-save counter (HS-32 blocks + ripple).
//
// Bins are staged per 64-feature chunk as 16-bit table byte offsets
// ((f*16 + b) * 4), two per 32-bit word, in a feature-major layout rotated by
// row so both the staging stores and the per-lane loads are bank-conflict
// free, and shared by the NC warps of a group.
//
// Work is scheduled dynamically in items = (block of rows, word slice), ordered
// block-major, so CTAs working concurrently on the same row block share its
// bins through L2 (each row's bins leave HBM ~once) while each CTA rebuilds
// its tables only when its slice changes (<1 % of an item's work).
#include <algorithm>

#include "hv_internal.cuh"

namespace hvb {

constexpr int kTBins = 16;    // table rows per feature (B <= 16)
constexpr int kChunk = 64;    // features per staged chunk
constexpr int kBlockRows = 8192;

struct TT2Params {
  const uint8_t* bins8;
  uint32_t ldb;
  uint64_t rows;
  uint32_t F, F16, D, W, B;
  const uint32_t* id;
  const uint32_t* val;
  const uint32_t* tie;
  uint32_t* out;
  uint32_t slices;       // ceil(W / NC)
  uint64_t blocks;       // ceil(rows / kBlockRows)
  unsigned int* counter;  // dynamic work counter (zeroed before launch)
};

// Harley–Seal over 32 inputs: acc[0..4] hold weights 1..16, the returned
// carry has weight 32.
template <int K, class Load>
__device__ __forceinline__ uint32_t hs_tree(uint32_t (&acc)[5], Load& ld) {
  if constexpr (K == 1) {
    const uint32_t a = ld();
    const uint32_t b = ld();
    uint32_t h;
    csa(h, acc[0], acc[0], a, b);
    return h;
  } else {
    const uint32_t c1 = hs_tree<K - 1>(acc, ld);
    const uint32_t c2 = hs_tree<K - 1>(acc, ld);
    uint32_t h;
    csa(h, acc[K - 1], acc[K - 1], c1, c2);
    return h;
  }
}

template <int NC, int G, int NH>
__global__ void __launch_bounds__(NC * G * 32, 2) encode_tt2_kernel(TT2Params p) {
  extern __shared__ __align__(16) uint32_t smem[];
  const uint32_t tsz = p.F16 * kTBins;  // words per table
  uint32_t* T = smem;                    // NC tables
  uint32_t* S = smem + NC * tsz;         // G x (32 pairs x 32 rows) offset words
  __shared__ unsigned int s_item;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int c = warp % NC;
  const int g = warp / NC;
  constexpr uint32_t nthreads = NC * G * 32;
  constexpr uint32_t tile_rows = 32u * G;
  const uint64_t items = static_cast<uint64_t>(p.slices) * p.blocks;
  const uint32_t nchunks = (p.F16 + kChunk - 1) / kChunk;
  uint32_t cur_slice = 0xFFFFFFFFu;
  const char* Tc = reinterpret_cast<const char*>(T + c * tsz);
  const uint32_t* Sg = S + g * (kChunk / 2) * 32;

  for (;;) {
    if (threadIdx.x == 0) s_item = atomicAdd(p.counter, 1u);
    __syncthreads();
    const uint64_t item = s_item;
    if (item >= items) break;
    const uint32_t slice = static_cast<uint32_t>(item % p.slices);
    const uint64_t block = item / p.slices;
    if (slice != cur_slice) {
      // T_cc[f][b] = ID_f[w] ^ V_b[w]; zero for f >= F, b >= B, w >= W
      for (uint32_t k = threadIdx.x; k < NC * tsz; k += nthreads) {
        const uint32_t cc = k / tsz;
        const uint32_t rem = k - cc * tsz;
        const uint32_t f = rem / kTBins;
        const uint32_t b = rem % kTBins;
        const uint32_t w = slice * NC + cc;
        uint32_t v = 0;
        if (w < p.W && f < p.F && b < p.B) {
          v = __ldg(p.id + static_cast<uint64_t>(f) * p.W + w) ^ __ldg(p.val + static_cast<uint64_t>(b) * p.W + w);
        }
        T[k] = v;
      }
      cur_slice = slice;
      __syncthreads();
    }
    const uint32_t w = slice * NC + c;
    const uint64_t r_begin = block * kBlockRows;
    const uint64_t r_end = min(p.rows, r_begin + kBlockRows);
    for (uint64_t tile0 = r_begin; tile0 < r_end; tile0 += tile_rows) {
      uint32_t acc[5] = {0, 0, 0, 0, 0};
      uint32_t hi[NH];
#pragma unroll
      for (int k = 0; k < NH; ++k) hi[k] = 0;
      for (uint32_t ch = 0; ch < nchunks; ++ch) {
        __syncthreads();
        // stage chunk ch: for every group, 32 rows x 64 features -> 32 offset
        // pairs per row, stored pair-major [pair][row] so that a warp's stores
        // (lane = row) and the per-lane loads below are both conflict free and
        // the loads need no address arithmetic (pair index is an immediate).
        // Each thread moves one full 32-byte sector (32 features) of one row.
        for (uint32_t k = threadIdx.x; k < G * 64; k += nthreads) {
          const uint32_t gg = k >> 6;
          const uint32_t hf = (k >> 5) & 1u;  // which 32-feature half of the chunk
          const uint32_t row = k & 31u;
          const uint64_t grow = tile0 + 32ull * gg + row;
          uint4 v0 = make_uint4(0, 0, 0, 0), v1 = v0;
          if (grow < r_end) {
            const uint4* src = reinterpret_cast<const uint4*>(p.bins8 + grow * p.ldb + ch * kChunk + hf * 32u);
            v0 = src[0];
            v1 = src[1];
          }
          const uint32_t words[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
          uint32_t* dst = S + gg * (kChunk / 2) * 32 + (hf * 16u) * 32 + row;
          const uint32_t fbase = (ch * kChunk + hf * 32u) * (kTBins * 4);
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            // byte offsets (f*16 + b)*4 of 4 features (f < F16 <= 1023 keeps them < 2^16)
            const uint32_t v = words[q];
            const uint32_t b0 = fbase + q * 256u;
            const uint32_t o0 = b0 + ((v & 0xFFu) << 2);
            const uint32_t o1 = b0 + 64u + (((v >> 8) & 0xFFu) << 2);
            const uint32_t o2 = b0 + 128u + (((v >> 16) & 0xFFu) << 2);
            const uint32_t o3 = b0 + 192u + ((v >> 24) << 2);
            dst[(2 * q) * 32] = o0 | (o1 << 16);
            dst[(2 * q + 1) * 32] = o2 | (o3 << 16);
          }
        }
        __syncthreads();
        const uint32_t nf = min(static_cast<uint32_t>(kChunk), p.F16 - ch * kChunk);  // multiple of 16
        uint32_t pair = 0;
        uint32_t cur = 0;
        int half = 0;
        auto ld = [&]() -> uint32_t {
          if (half == 0) {
            cur = Sg[pair * 32 + lane];
            ++pair;
          }
          const uint32_t off = half ? (cur >> 16) : (cur & 0xFFFFu);
          half ^= 1;
          return *reinterpret_cast<const uint32_t*>(Tc + off);
        };
        if (nf == kChunk) {
#pragma unroll
          for (int h32 = 0; h32 < 2; ++h32) {
            uint32_t carry = hs_tree<5>(acc, ld);
#pragma unroll
            for (int k = 0; k < NH; ++k) {
              const uint32_t t = hi[k] & carry;
              hi[k] ^= carry;
              carry = t;
            }
          }
        } else {
          // tail: blocks of 16 features, carry of weight 16 rippled from acc[4]
          for (uint32_t f16 = 0; f16 < nf; f16 += 16) {
            uint32_t carry = hs_tree<4>(acc, ld);
            const uint32_t t = acc[4] & carry;
            acc[4] ^= carry;
            carry = t;
#pragma unroll
            for (int k = 0; k < NH; ++k) {
              const uint32_t u = hi[k] & carry;
              hi[k] ^= carry;
              carry = u;
            }
          }
        }
      }
      // majority against F: bit = 2c > F ? 1 : 2c < F ? 0 : tie (planes: acc[0..4], hi[0..NH))
      const uint64_t row = tile0 + 32ull * g + lane;
      if (w < p.W && row < r_end) {
        const uint32_t half_f = p.F >> 1;
        uint32_t gt = 0u, eq = 0xFFFFFFFFu;
#pragma unroll
        for (int k = 4 + NH; k >= 0; --k) {
          const uint32_t pl = k >= 5 ? hi[k - 5] : acc[k];
          if ((half_f >> k) & 1u) {
            eq &= pl;
          } else {
            gt |= eq & pl;
            eq &= ~pl;
          }
        }
        const uint32_t bit = gt | ((p.F & 1u) ? 0u : (eq & __ldg(p.tie + w)));
        p.out[row * p.W + w] = bit & valid_mask(w, p.D);
      }
    }
  }
}

namespace {

template <int NC, int G, int NH>
void launch_tt2_inst(hv_context* ctx, cudaStream_t st, TT2Params p, size_t smem) {
  auto kern = encode_tt2_kernel<NC, G, NH>;
  ck(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)),
     "cudaFuncSetAttribute");
  int per_sm = 0;
  ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NC * G * 32, smem), "occupancy");
  if (per_sm < 1) fail(HV_ERR_CUDA, "encode_tt2_kernel: configuration does not fit on an SM");
  const uint64_t items = static_cast<uint64_t>(p.slices) * p.blocks;
  const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(items, static_cast<uint64_t>(ctx->sm_count) * per_sm));
  ck(cudaMemsetAsync(p.counter, 0, sizeof(unsigned int), st), "counter reset");
  kern<<<grid, NC * G * 32, smem, st>>>(p);
  launched("encode_tt2_kernel");
}

}  // namespace

bool launch_tt(hv_context* ctx, cudaStream_t st, const uint8_t* bins8, uint32_t ldb, uint64_t rows, uint32_t F,
               const uint32_t* id, const uint32_t* val, uint32_t B, uint32_t D, uint32_t W, const uint32_t* tie,
               uint32_t* out) {
  if (B > static_cast<uint32_t>(kTBins) || F == 0 || rows == 0) return false;
  if (ldb % kChunk != 0 || (reinterpret_cast<uintptr_t>(bins8) & 15u)) return false;
  const uint32_t F16 = (F + 15) / 16 * 16;
  if (static_cast<uint64_t>(F16) * kTBins * 4 > 0xFFFF) return false;  // 16-bit table offsets
  // planes beyond the 5 HS levels: counts < 32 * 2^NH
  int nh = 1;
  while ((32ull << nh) <= F) ++nh;
  if (nh > 5) return false;
  const size_t table = static_cast<size_t>(F16) * kTBins * 4;
  const size_t stage = static_cast<size_t>(kChunk / 2) * 32 * 4;  // per group
  const size_t per_sm_smem = 227 * 1024;
  // prefer the widest slice that still fits two CTAs per SM, else one CTA
  struct Shape { int nc, g; };
  const Shape shapes[] = {{4, 4}, {2, 8}, {1, 16}};
  int pick = -1;
  for (int pass = 0; pass < 2 && pick < 0; ++pass) {
    for (int i = 0; i < 3; ++i) {
      const size_t smem = shapes[i].nc * table + shapes[i].g * stage;
      const size_t limit = pass == 0 ? per_sm_smem / 2 - 2048 : std::min<size_t>(ctx->smem_optin, per_sm_smem - 2048);
      if (smem <= limit) {
        pick = i;
        break;
      }
    }
  }
  if (pick < 0) return false;
  const Shape s = shapes[pick];
  const size_t smem = s.nc * table + s.g * stage;
  // one work counter per launch from the context's ring (concurrent launches on
  // the context's two streams must not share one)
  unsigned int* counter = ctx->d_counters + (ctx->next_counter++ % hv_context::kCounters);
  TT2Params p{bins8, ldb, rows, F, F16, D, W, B, id, val, tie, out,
              static_cast<uint32_t>((W + s.nc - 1) / s.nc), (rows + kBlockRows - 1) / kBlockRows, counter};
#define HV_TT2(NC, G, N)                                  \
  if (s.nc == NC && nh == N) {                            \
    launch_tt2_inst<NC, G, N>(ctx, st, p, smem);          \
    return true;                                          \
  }
#define HV_TT2_NH(NC, G) HV_TT2(NC, G, 1) HV_TT2(NC, G, 2) HV_TT2(NC, G, 3) HV_TT2(NC, G, 4) HV_TT2(NC, G, 5)
  HV_TT2_NH(4, 4)
  HV_TT2_NH(2, 8)
  HV_TT2_NH(1, 16)
#undef HV_TT2_NH
#undef HV_TT2
  return false;
}

}  // namespace hvb
