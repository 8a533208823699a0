// hv_encode_tt.cu — the fast ID-level encoder (reference encoding.cpp:266-272,
// the hot loop of the whole pipeline).
//
// Output bit j of datapoint i = majority over f < F of ID_f[j] ^ V_{bin(i,f)}[j].
// Per CTA, shared memory holds, for NP pairs of output words (w0, w1),
//     T_p[f][b] = { ID_f[w0] ^ V_b[w0], ID_f[w1] ^ V_b[w1] }   (8 bytes)
// so the XOR bind disappears and one 64-bit LDS yields the bound words of two
// output words. Lane = datapoint; warp (p, g) = word pair p for the 32
// datapoints of group g. The 16 bins of one feature occupy 128 contiguous bytes,
// so each half-warp's LDS.64 is bank-conflict free for any bin pattern (equal
// bins broadcast). Per lane and bound word the cost is half an LDS.64, half a
// byte extract (PRMT) and a ~2.2-LOP3 share of a bit-sliced Harley–Seal
// carry-save counter (HS-32 blocks + ripple into the high planes).
//
// Raw uint8 bins are staged per 64-feature chunk in a [word][row] layout (lane
// = row on both the stores and the loads: conflict free, no address math),
// double-buffered through registers so the global loads of chunk k+1 overlap
// the counting of chunk k, with one CTA barrier per chunk.
//
// Work is scheduled dynamically in items = (block of rows, word-pair slice),
// ordered block-major, so CTAs working concurrently on the same row block share
// its bins through L2 (each row's bins leave HBM ~once) while each CTA rebuilds
// its tables only when its slice changes.
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "hv_internal.cuh"

namespace hvb {

constexpr int kTBins = 16;     // table rows per feature (B <= 16)
constexpr int kChunk = 64;     // features per staged chunk
constexpr int kBlockRows = 8192;

struct TT3Params {
  const uint8_t* bins8;
  uint32_t ldb;
  uint64_t rows;
  uint32_t F, F16, D, W, B;
  const uint32_t* id;
  const uint32_t* val;
  const uint32_t* tie;
  uint32_t* out;
  uint32_t slices;        // ceil(W / (2 NP))
  uint64_t blocks;        // ceil(rows / kBlockRows)
  unsigned int* counter;  // dynamic work counter (zeroed before launch)
};

struct HS2 {
  uint32_t a[5], b[5];
};

// Harley–Seal over 2^K inputs for two independent counters (word pair).
// Levels 0..K-1 accumulate; the returned carries have weight 2^K.
template <int K, class Load>
__device__ __forceinline__ uint2 hs_tree2(HS2& s, Load& ld) {
  if constexpr (K == 1) {
    const uint2 x = ld();
    const uint2 y = ld();
    uint2 h;
    csa(h.x, s.a[0], s.a[0], x.x, y.x);
    csa(h.y, s.b[0], s.b[0], x.y, y.y);
    return h;
  } else {
    const uint2 c1 = hs_tree2<K - 1>(s, ld);
    const uint2 c2 = hs_tree2<K - 1>(s, ld);
    uint2 h;
    csa(h.x, s.a[K - 1], s.a[K - 1], c1.x, c2.x);
    csa(h.y, s.b[K - 1], s.b[K - 1], c1.y, c2.y);
    return h;
  }
}

template <int NH>
__device__ __forceinline__ void ripple(uint32_t (&hi)[NH], uint32_t carry) {
#pragma unroll
  for (int k = 0; k < NH; ++k) {
    const uint32_t t = hi[k] & carry;
    hi[k] ^= carry;
    carry = t;
  }
}

// bit = 2c > F ? 1 : 2c < F ? 0 : tie   (planes acc[0..4] weights 1..16, hi[k] weight 32 << k)
template <int NH>
__device__ __forceinline__ uint32_t majority_bits(const uint32_t (&acc)[5], const uint32_t (&hi)[NH], uint32_t F,
                                                  uint32_t tie) {
  const uint32_t half_f = F >> 1;
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
  return gt | ((F & 1u) ? 0u : (eq & tie));
}

template <int NP, int G, int NH>
__global__ void __launch_bounds__(NP * G * 32, 2) encode_tt3_kernel(TT3Params p) {
  extern __shared__ __align__(16) uint32_t smem[];
  const uint32_t tsz = p.F16 * kTBins * 2;  // words per pair table
  uint32_t* T = smem;                        // NP tables of uint2 entries
  uint32_t* S = smem + NP * tsz;             // 2 buffers x G groups x 16 words x 32 rows
  constexpr uint32_t kStage = 16 * 32;       // words per group and buffer
  __shared__ unsigned int s_item;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int cp = warp % NP;
  const int g = warp / NP;
  constexpr uint32_t nthreads = NP * G * 32;
  constexpr uint32_t tile_rows = 32u * G;
  const uint64_t items = static_cast<uint64_t>(p.slices) * p.blocks;
  const uint32_t nchunks = (p.F16 + kChunk - 1) / kChunk;
  uint32_t cur_slice = 0xFFFFFFFFu;
  const char* Tp = reinterpret_cast<const char*>(T + cp * tsz);

  // staging role: per chunk, G*64 32-byte sectors (group, half, row); thread
  // owns sectors threadIdx.x + i*nthreads, i < SPT.
  constexpr int SPT = (G * 64 + nthreads - 1) / nthreads;

  for (;;) {
    if (threadIdx.x == 0) s_item = atomicAdd(p.counter, 1u);
    __syncthreads();
    const uint64_t item = s_item;
    if (item >= items) break;
    const uint32_t slice = static_cast<uint32_t>(item % p.slices);
    const uint64_t block = item / p.slices;
    if (slice != cur_slice) {
      // T_pp[f][b] = {ID_f[w0]^V_b[w0], ID_f[w1]^V_b[w1]}; zero for f >= F, b >= B, w >= W
      for (uint32_t k = threadIdx.x; k < NP * tsz; k += nthreads) {
        const uint32_t pp = k / tsz;
        const uint32_t rem = k - pp * tsz;
        const uint32_t f = rem / (kTBins * 2);
        const uint32_t b = (rem / 2) % kTBins;
        const uint32_t w = 2 * (slice * NP + pp) + (rem & 1u);
        uint32_t v = 0;
        if (w < p.W && f < p.F && b < p.B) {
          v = __ldg(p.id + static_cast<uint64_t>(f) * p.W + w) ^ __ldg(p.val + static_cast<uint64_t>(b) * p.W + w);
        }
        T[k] = v;
      }
      cur_slice = slice;
      __syncthreads();
    }
    const uint32_t w0 = 2 * (slice * NP + cp);
    const uint64_t r_begin = block * kBlockRows;
    const uint64_t r_end = min(p.rows, r_begin + kBlockRows);
    for (uint64_t tile0 = r_begin; tile0 < r_end; tile0 += tile_rows) {
      HS2 s;
#pragma unroll
      for (int k = 0; k < 5; ++k) s.a[k] = s.b[k] = 0;
      uint32_t hia[NH], hib[NH];
#pragma unroll
      for (int k = 0; k < NH; ++k) hia[k] = hib[k] = 0;

      // prefetch chunk 0 into registers, store, barrier
      const uint4* st_src[SPT];
      bool st_valid[SPT];
      uint32_t* st_dst[SPT];
      uint4 r0[SPT], r1[SPT];
#pragma unroll
      for (int i = 0; i < SPT; ++i) {
        const uint32_t k = threadIdx.x + i * nthreads;
        const uint32_t sg = k >> 6, sh = (k >> 5) & 1u, sr = k & 31u;
        const uint64_t grow = tile0 + 32ull * sg + sr;
        st_valid[i] = k < G * 64u && grow < r_end;
        st_src[i] = reinterpret_cast<const uint4*>(p.bins8 + (st_valid[i] ? grow : 0) * p.ldb + sh * 32u);
        st_dst[i] = S + (k < G * 64u ? sg : 0) * kStage + (sh * 8u) * 32 + sr;
        r0[i] = r1[i] = make_uint4(0, 0, 0, 0);
        if (st_valid[i]) {
          r0[i] = st_src[i][0];
          r1[i] = st_src[i][1];
        }
      }
      auto stage = [&](uint32_t buf) {
#pragma unroll
        for (int i = 0; i < SPT; ++i) {
          if (threadIdx.x + i * nthreads < G * 64u) {
            uint32_t* dst = st_dst[i] + buf * G * kStage;
            dst[0 * 32] = r0[i].x;
            dst[1 * 32] = r0[i].y;
            dst[2 * 32] = r0[i].z;
            dst[3 * 32] = r0[i].w;
            dst[4 * 32] = r1[i].x;
            dst[5 * 32] = r1[i].y;
            dst[6 * 32] = r1[i].z;
            dst[7 * 32] = r1[i].w;
          }
        }
      };
      stage(0);  // buffer 0 is free: the previous tile ended with a barrier
      __syncthreads();
      for (uint32_t ch = 0; ch < nchunks; ++ch) {
        const uint32_t buf = ch & 1u;
        const bool more = ch + 1 < nchunks;
        if (more) {  // issue the next chunk's loads; they land during the counting below
#pragma unroll
          for (int i = 0; i < SPT; ++i) {
            if (st_valid[i]) {
              r0[i] = st_src[i][(ch + 1) * (kChunk / 16)];
              r1[i] = st_src[i][(ch + 1) * (kChunk / 16) + 1];
            }
          }
        }
        const uint32_t* Sg = S + (buf * G + g) * kStage;
        const char* Tch = Tp + static_cast<size_t>(ch) * kChunk * kTBins * 8;
        const uint32_t nf = min(static_cast<uint32_t>(kChunk), p.F16 - ch * kChunk);  // multiple of 16
        uint32_t q = 0, word = 0;
        int t = 0;
        auto ld = [&]() -> uint2 {
          if (t == 0) word = Sg[q * 32 + lane];
          const uint32_t b = __byte_perm(word, 0, 0x4440 | t);
          const uint2 v = *reinterpret_cast<const uint2*>(Tch + (q * 4 + t) * (kTBins * 8) + b * 8);
          if (++t == 4) {
            t = 0;
            ++q;
          }
          return v;
        };
        if (nf == kChunk) {
#pragma unroll
          for (int h32 = 0; h32 < 2; ++h32) {
            const uint2 carry = hs_tree2<5>(s, ld);
            ripple<NH>(hia, carry.x);
            ripple<NH>(hib, carry.y);
          }
        } else {
          for (uint32_t f16 = 0; f16 < nf; f16 += 16) {
            uint2 carry = hs_tree2<4>(s, ld);
            const uint32_t ta = s.a[4] & carry.x, tb = s.b[4] & carry.y;
            s.a[4] ^= carry.x;
            s.b[4] ^= carry.y;
            ripple<NH>(hia, ta);
            ripple<NH>(hib, tb);
          }
        }
        if (more) stage(buf ^ 1u);
        __syncthreads();
      }
      const uint64_t row = tile0 + 32ull * g + lane;
      if (row < r_end) {
        uint32_t* o = p.out + row * p.W;
        if (w0 < p.W) o[w0] = majority_bits<NH>(s.a, hia, p.F, __ldg(p.tie + w0)) & valid_mask(w0, p.D);
        if (w0 + 1 < p.W) o[w0 + 1] = majority_bits<NH>(s.b, hib, p.F, __ldg(p.tie + w0 + 1)) & valid_mask(w0 + 1, p.D);
      }
    }
  }
}

// v4: same tables and counters as v3, but every lane streams its own row's
// bins straight into registers (64 bytes per chunk, next chunk prefetched while
// the current one is counted) — no shared staging, no CTA barrier per chunk;
// warps of a CTA only meet at table rebuilds.
template <int NP, int G, int NH>
__global__ void __launch_bounds__(NP * G * 32, 2) encode_tt4_kernel(TT3Params p) {
  extern __shared__ __align__(16) uint32_t smem[];
  const uint32_t tsz = p.F16 * kTBins * 2;  // words per pair table
  uint32_t* T = smem;                        // NP tables of uint2 entries
  __shared__ unsigned int s_item;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int cp = warp % NP;
  const int g = warp / NP;
  constexpr uint32_t nthreads = NP * G * 32;
  constexpr uint32_t tile_rows = 32u * G;
  const uint64_t items = static_cast<uint64_t>(p.slices) * p.blocks;
  const uint32_t nchunks = (p.F16 + kChunk - 1) / kChunk;
  uint32_t cur_slice = 0xFFFFFFFFu;
  const char* Tp = reinterpret_cast<const char*>(T + cp * tsz);

  for (;;) {
    if (threadIdx.x == 0) s_item = atomicAdd(p.counter, 1u);
    __syncthreads();
    const uint64_t item = s_item;
    __syncthreads();  // everyone has read s_item before thread 0 can overwrite it
    if (item >= items) break;
    const uint32_t slice = static_cast<uint32_t>(item % p.slices);
    const uint64_t block = item / p.slices;
    if (slice != cur_slice) {
      for (uint32_t k = threadIdx.x; k < NP * tsz; k += nthreads) {
        const uint32_t pp = k / tsz;
        const uint32_t rem = k - pp * tsz;
        const uint32_t f = rem / (kTBins * 2);
        const uint32_t b = (rem / 2) % kTBins;
        const uint32_t w = 2 * (slice * NP + pp) + (rem & 1u);
        uint32_t v = 0;
        if (w < p.W && f < p.F && b < p.B) {
          v = __ldg(p.id + static_cast<uint64_t>(f) * p.W + w) ^ __ldg(p.val + static_cast<uint64_t>(b) * p.W + w);
        }
        T[k] = v;
      }
      cur_slice = slice;
      __syncthreads();
    }
    const uint32_t w0 = 2 * (slice * NP + cp);
    const uint64_t r_begin = block * kBlockRows;
    const uint64_t r_end = min(p.rows, r_begin + kBlockRows);
    for (uint64_t tile0 = r_begin; tile0 < r_end; tile0 += tile_rows) {
      const uint64_t row = tile0 + 32ull * g + lane;
      const bool valid = row < r_end;
      const uint4* src = reinterpret_cast<const uint4*>(p.bins8 + (valid ? row : 0) * p.ldb);
      HS2 s;
#pragma unroll
      for (int k = 0; k < 5; ++k) s.a[k] = s.b[k] = 0;
      uint32_t hia[NH], hib[NH];
#pragma unroll
      for (int k = 0; k < NH; ++k) hia[k] = hib[k] = 0;
      uint4 cur[4], nxt[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) cur[k] = valid ? __ldg(src + k) : make_uint4(0, 0, 0, 0);
      for (uint32_t ch = 0; ch < nchunks; ++ch) {
        if (ch + 1 < nchunks) {
#pragma unroll
          for (int k = 0; k < 4; ++k) nxt[k] = valid ? __ldg(src + (ch + 1) * (kChunk / 16) + k) : make_uint4(0, 0, 0, 0);
        }
        const uint32_t bw[16] = {cur[0].x, cur[0].y, cur[0].z, cur[0].w, cur[1].x, cur[1].y, cur[1].z, cur[1].w,
                                 cur[2].x, cur[2].y, cur[2].z, cur[2].w, cur[3].x, cur[3].y, cur[3].z, cur[3].w};
        const char* Tch = Tp + static_cast<size_t>(ch) * kChunk * kTBins * 8;
        int i = 0;
        auto ld = [&]() -> uint2 {
          const uint32_t b = __byte_perm(bw[i >> 2], 0, 0x4440 | (i & 3));
          const uint2 v = *reinterpret_cast<const uint2*>(Tch + i * (kTBins * 8) + b * 8);
          ++i;
          return v;
        };
        const uint32_t nf = min(static_cast<uint32_t>(kChunk), p.F16 - ch * kChunk);  // multiple of 16
        if (nf == kChunk) {
#pragma unroll
          for (int h32 = 0; h32 < 2; ++h32) {
            const uint2 carry = hs_tree2<5>(s, ld);
            ripple<NH>(hia, carry.x);
            ripple<NH>(hib, carry.y);
          }
        } else {
          // 1..3 tail blocks of 16 features; carries of weight 16 enter at level 4
          auto block16 = [&]() {
            const uint2 carry = hs_tree2<4>(s, ld);
            const uint32_t ta = s.a[4] & carry.x, tb = s.b[4] & carry.y;
            s.a[4] ^= carry.x;
            s.b[4] ^= carry.y;
            ripple<NH>(hia, ta);
            ripple<NH>(hib, tb);
          };
          block16();
          if (nf > 16) block16();
          if (nf > 32) block16();
        }
        if (ch + 1 < nchunks) {
#pragma unroll
          for (int k = 0; k < 4; ++k) cur[k] = nxt[k];
        }
      }
      if (valid) {
        uint32_t* o = p.out + row * p.W;
        if (w0 < p.W) o[w0] = majority_bits<NH>(s.a, hia, p.F, __ldg(p.tie + w0)) & valid_mask(w0, p.D);
        if (w0 + 1 < p.W) o[w0 + 1] = majority_bits<NH>(s.b, hib, p.F, __ldg(p.tie + w0 + 1)) & valid_mask(w0 + 1, p.D);
      }
    }
  }
}

// v5: like v4 (no CTA barriers, warps independent), but each warp loads its 32
// rows' chunk coalesced (4 lanes per 64-byte row -> 8 lines per request
// instead of 32) and transposes it through a private, double-buffered
// shared-memory buffer. Word w of row r lives at [w][r ^ 8*(w>>2)]: the 16
// stores and 16 loads per lane and chunk are bank-conflict free and the loads
// use 4 precomputed lane bases with immediate offsets.
template <int NP, int G, int NH>
__global__ void __launch_bounds__(NP * G * 32, 2) encode_tt5_kernel(TT3Params p) {
  extern __shared__ __align__(16) uint32_t smem[];
  const uint32_t tsz = p.F16 * kTBins * 2;  // words per pair table
  uint32_t* T = smem;                        // NP tables of uint2 entries
  __shared__ unsigned int s_item;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int cp = warp % NP;
  const int g = warp / NP;
  constexpr uint32_t nthreads = NP * G * 32;
  constexpr uint32_t tile_rows = 32u * G;
  uint32_t* Sw = smem + NP * tsz + warp * (2 * 16 * 32);  // private double buffer [buf][16 words][32 rows]
  const uint64_t items = static_cast<uint64_t>(p.slices) * p.blocks;
  const uint32_t nchunks = (p.F16 + kChunk - 1) / kChunk;
  uint32_t cur_slice = 0xFFFFFFFFu;
  const char* Tp = reinterpret_cast<const char*>(T + cp * tsz);
  // loader role: lane -> (row sub-index lr = lane/4, quad q = lane%4); request i covers rows 8i..8i+7
  const uint32_t lr = lane >> 2, lq = lane & 3u;

  for (;;) {
    if (threadIdx.x == 0) s_item = atomicAdd(p.counter, 1u);
    __syncthreads();
    const uint64_t item = s_item;
    __syncthreads();
    if (item >= items) break;
    const uint32_t slice = static_cast<uint32_t>(item % p.slices);
    const uint64_t block = item / p.slices;
    if (slice != cur_slice) {
      for (uint32_t k = threadIdx.x; k < NP * tsz; k += nthreads) {
        const uint32_t pp = k / tsz;
        const uint32_t rem = k - pp * tsz;
        const uint32_t f = rem / (kTBins * 2);
        const uint32_t b = (rem / 2) % kTBins;
        const uint32_t w = 2 * (slice * NP + pp) + (rem & 1u);
        uint32_t v = 0;
        if (w < p.W && f < p.F && b < p.B) {
          v = __ldg(p.id + static_cast<uint64_t>(f) * p.W + w) ^ __ldg(p.val + static_cast<uint64_t>(b) * p.W + w);
        }
        T[k] = v;
      }
      cur_slice = slice;
      __syncthreads();
    }
    const uint32_t w0 = 2 * (slice * NP + cp);
    const uint64_t r_begin = block * kBlockRows;
    const uint64_t r_end = min(p.rows, r_begin + kBlockRows);
    for (uint64_t tile0 = r_begin; tile0 < r_end; tile0 += tile_rows) {
      const uint64_t wrow0 = tile0 + 32ull * g;  // this warp's 32 rows
      HS2 s;
#pragma unroll
      for (int k = 0; k < 5; ++k) s.a[k] = s.b[k] = 0;
      uint32_t hia[NH], hib[NH];
#pragma unroll
      for (int k = 0; k < NH; ++k) hia[k] = hib[k] = 0;
      // coalesced loads of the chunk: request i -> row 8i + lr, bytes 16*lq .. 16*lq+15
      const uint4* src[4];
      bool ok[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint64_t r = wrow0 + 8 * i + lr;
        ok[i] = r < r_end;
        src[i] = reinterpret_cast<const uint4*>(p.bins8 + (ok[i] ? r : 0) * p.ldb) + lq;
      }
      uint4 ld4[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) ld4[i] = ok[i] ? __ldg(src[i]) : make_uint4(0, 0, 0, 0);
      auto stage = [&](uint32_t buf) {
        uint32_t* B = Sw + buf * (16 * 32);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const uint32_t r = 8 * i + lr;
          const uint32_t col = r ^ (lq << 3);  // words 4lq..4lq+3 share w>>2 = lq
          B[(4 * lq + 0) * 32 + col] = ld4[i].x;
          B[(4 * lq + 1) * 32 + col] = ld4[i].y;
          B[(4 * lq + 2) * 32 + col] = ld4[i].z;
          B[(4 * lq + 3) * 32 + col] = ld4[i].w;
        }
      };
      stage(0);
      __syncwarp();
      for (uint32_t ch = 0; ch < nchunks; ++ch) {
        const uint32_t buf = ch & 1u;
        const bool more = ch + 1 < nchunks;
        if (more) {
#pragma unroll
          for (int i = 0; i < 4; ++i) ld4[i] = ok[i] ? __ldg(src[i] + (ch + 1) * (kChunk / 16)) : make_uint4(0, 0, 0, 0);
        }
        const uint32_t* B = Sw + buf * (16 * 32);
        const uint32_t* base[4] = {B + (lane ^ 0), B + (lane ^ 8), B + (lane ^ 16), B + (lane ^ 24)};
        const char* Tch = Tp + static_cast<size_t>(ch) * kChunk * kTBins * 8;
        int i = 0;
        uint32_t word = 0;
        auto ld = [&]() -> uint2 {
          if ((i & 3) == 0) word = base[(i >> 4) & 3][(i >> 2) * 32];
          const uint32_t b = __byte_perm(word, 0, 0x4440 | (i & 3));
          const uint2 v = *reinterpret_cast<const uint2*>(Tch + i * (kTBins * 8) + b * 8);
          ++i;
          return v;
        };
        const uint32_t nf = min(static_cast<uint32_t>(kChunk), p.F16 - ch * kChunk);  // multiple of 16
        if (nf == kChunk) {
#pragma unroll
          for (int h32 = 0; h32 < 2; ++h32) {
            const uint2 carry = hs_tree2<5>(s, ld);
            ripple<NH>(hia, carry.x);
            ripple<NH>(hib, carry.y);
          }
        } else {
          auto block16 = [&]() {
            const uint2 carry = hs_tree2<4>(s, ld);
            const uint32_t ta = s.a[4] & carry.x, tb = s.b[4] & carry.y;
            s.a[4] ^= carry.x;
            s.b[4] ^= carry.y;
            ripple<NH>(hia, ta);
            ripple<NH>(hib, tb);
          };
          block16();
          if (nf > 16) block16();
          if (nf > 32) block16();
        }
        if (more) {
          stage(buf ^ 1u);  // other buffer: its last readers finished before the previous __syncwarp
          __syncwarp();
        }
      }
      const uint64_t row = wrow0 + lane;
      if (row < r_end) {
        uint32_t* o = p.out + row * p.W;
        if (w0 < p.W) o[w0] = majority_bits<NH>(s.a, hia, p.F, __ldg(p.tie + w0)) & valid_mask(w0, p.D);
        if (w0 + 1 < p.W) o[w0 + 1] = majority_bits<NH>(s.b, hib, p.F, __ldg(p.tie + w0 + 1)) & valid_mask(w0 + 1, p.D);
      }
      __syncwarp();  // buffer 0 of the next tile is rewritten next
    }
  }
}

namespace {

template <int NP, int G, int NH>
void launch_tt5_inst(hv_context* ctx, cudaStream_t st, TT3Params p, size_t smem) {
  auto kern = encode_tt5_kernel<NP, G, NH>;
  ck(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)),
     "cudaFuncSetAttribute");
  int per_sm = 0;
  ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NP * G * 32, smem), "occupancy");
  if (per_sm < 1) fail(HV_ERR_CUDA, "encode_tt5_kernel: configuration does not fit on an SM");
  const uint64_t items = static_cast<uint64_t>(p.slices) * p.blocks;
  const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(items, static_cast<uint64_t>(ctx->sm_count) * per_sm));
  ck(cudaMemsetAsync(p.counter, 0, sizeof(unsigned int), st), "counter reset");
  kern<<<grid, NP * G * 32, smem, st>>>(p);
  launched("encode_tt5_kernel");
}

template <int NP, int G, int NH>
void launch_tt4_inst(hv_context* ctx, cudaStream_t st, TT3Params p, size_t smem) {
  auto kern = encode_tt4_kernel<NP, G, NH>;
  ck(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)),
     "cudaFuncSetAttribute");
  int per_sm = 0;
  ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NP * G * 32, smem), "occupancy");
  if (per_sm < 1) fail(HV_ERR_CUDA, "encode_tt4_kernel: configuration does not fit on an SM");
  const uint64_t items = static_cast<uint64_t>(p.slices) * p.blocks;
  const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(items, static_cast<uint64_t>(ctx->sm_count) * per_sm));
  ck(cudaMemsetAsync(p.counter, 0, sizeof(unsigned int), st), "counter reset");
  kern<<<grid, NP * G * 32, smem, st>>>(p);
  launched("encode_tt4_kernel");
}

template <int NP, int G, int NH>
void launch_tt3_inst(hv_context* ctx, cudaStream_t st, TT3Params p, size_t smem) {
  auto kern = encode_tt3_kernel<NP, G, NH>;
  ck(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)),
     "cudaFuncSetAttribute");
  int per_sm = 0;
  ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NP * G * 32, smem), "occupancy");
  if (per_sm < 1) fail(HV_ERR_CUDA, "encode_tt3_kernel: configuration does not fit on an SM");
  const uint64_t items = static_cast<uint64_t>(p.slices) * p.blocks;
  const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(items, static_cast<uint64_t>(ctx->sm_count) * per_sm));
  ck(cudaMemsetAsync(p.counter, 0, sizeof(unsigned int), st), "counter reset");
  kern<<<grid, NP * G * 32, smem, st>>>(p);
  launched("encode_tt3_kernel");
}

}  // namespace

bool launch_tt(hv_context* ctx, cudaStream_t st, const uint8_t* bins8, uint32_t ldb, uint64_t rows, uint32_t F,
               const uint32_t* id, const uint32_t* val, uint32_t B, uint32_t D, uint32_t W, const uint32_t* tie,
               uint32_t* out) {
  if (B > static_cast<uint32_t>(kTBins) || F == 0 || rows == 0) return false;
  if (ldb % kChunk != 0 || (reinterpret_cast<uintptr_t>(bins8) & 15u)) return false;
  const uint32_t F16 = (F + 15) / 16 * 16;
  // planes beyond the 5 HS levels: counts < 32 * 2^NH
  int nh = 1;
  while ((32ull << nh) <= F) ++nh;
  if (nh > 6) return false;
  const size_t table = static_cast<size_t>(F16) * kTBins * 8;
  const char* ver_env = getenv("HVB200_TT_VERSION");
  const int version = ver_env ? atoi(ver_env) : 5;
  // v3 stages bins in shared memory (double-buffered, per row group); v4 keeps
  // them in registers and needs only the tables.
  const size_t stage = version == 3 ? 2ull * 16 * 32 * 4 : 0;  // per row group
  const size_t wstage = version == 5 ? 2ull * 16 * 32 * 4 : 0;  // per warp (private)
  // Shapes (word pairs x row groups), best measured first; the first two are
  // used when two CTAs fit on an SM.
  struct Shape { int np, g; };
  const Shape shapes[] = {{1, 8}, {2, 4}, {2, 8}, {1, 16}};
  const size_t two = 113 * 1024, one = std::min<size_t>(ctx->smem_optin, 225 * 1024);
  int pick = -1;
  for (int i = 0; i < 4 && pick < 0; ++i) {
    if (shapes[i].np * table + shapes[i].g * stage + shapes[i].np * shapes[i].g * wstage <= (i < 2 ? two : one)) {
      pick = i;
    }
  }
  if (const char* env = getenv("HVB200_TT_SHAPE")) {  // tuning override "np,g"
    int np = 0, g = 0;
    if (sscanf(env, "%d,%d", &np, &g) == 2) {
      for (int i = 0; i < 4; ++i) {
        if (shapes[i].np == np && shapes[i].g == g && np * table + g * stage + np * g * wstage <= one) pick = i;
      }
    }
  }
  if (pick < 0) return false;
  const Shape s = shapes[pick];
  const size_t smem = s.np * table + s.g * stage + s.np * s.g * wstage;
  // one work counter per launch from the context's ring (concurrent launches on
  // the context's two streams must not share one)
  unsigned int* counter = ctx->d_counters + (ctx->next_counter++ % hv_context::kCounters);
  TT3Params p{bins8, ldb, rows, F, F16, D, W, B, id, val, tie, out,
              static_cast<uint32_t>((W + 2 * s.np - 1) / (2 * s.np)), (rows + kBlockRows - 1) / kBlockRows, counter};
#define HV_TT(V, NP, G, N)                                   \
  if (version == V && s.np == NP && s.g == G && nh == N) {   \
    launch_tt##V##_inst<NP, G, N>(ctx, st, p, smem);         \
    return true;                                             \
  }
#define HV_TT_NH(V, NP, G) HV_TT(V, NP, G, 1) HV_TT(V, NP, G, 2) HV_TT(V, NP, G, 3) HV_TT(V, NP, G, 4) \
                           HV_TT(V, NP, G, 5) HV_TT(V, NP, G, 6)
  HV_TT_NH(5, 1, 8)
  HV_TT_NH(5, 2, 4)
  HV_TT_NH(5, 2, 8)
  HV_TT_NH(5, 1, 16)
  HV_TT_NH(4, 2, 4)
  HV_TT_NH(4, 1, 8)
  HV_TT_NH(4, 2, 8)
  HV_TT_NH(4, 1, 16)
  HV_TT_NH(3, 2, 4)
  HV_TT_NH(3, 1, 8)
  HV_TT_NH(3, 2, 8)
  HV_TT_NH(3, 1, 16)
#undef HV_TT_NH
#undef HV_TT
  return false;
}

}  // namespace hvb
