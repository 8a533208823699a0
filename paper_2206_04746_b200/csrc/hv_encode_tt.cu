// hv_encode_tt.cu — the fast ID-level encoder (reference encoding.cpp:266-272,
// the hot loop of the whole pipeline).
//
// Output bit j of datapoint i = majority over f < F of ID_f[j] ^ V_{bin(i,f)}[j].
// Lane = datapoint. Each CTA keeps, in shared memory, the bound words of NW =
// 2*NPR consecutive output words for every (feature, bin):
//     T[f][t][b] = { ID_f[w_2t] ^ V_b[w_2t], ID_f[w_2t+1] ^ V_b[w_2t+1] }   (8 B)
// so the XOR bind disappears into the table and a bound word costs exactly
// 4 bytes of shared-memory traffic: the 16 bins of (f, t) occupy 128
// contiguous bytes, so each half-warp's LDS.64 is bank-conflict free for any
// bin pattern. The table address is one byte permute (bins are staged
// pre-scaled by 8, PRMT splices the byte into the 256-aligned chunk base) and
// the per-pair offsets are immediates. Counting is a bit-sliced Harley–Seal
// carry-save tree over 64 features (2 LOP3 per bound word) rippling into the
// high planes once per 64 features; the counter starts biased so that the
// majority is its top plane (majority_biased).
//
// Binding ceilings per SM and clock: shared memory delivers 32 bound words
// (128 B), the ALU pipe 64 LOP3 = 32 bound words — both are saturated
// together, which is why the table entries are as wide as possible (NPR pairs
// share one PRMT and one bin staging) and nothing else runs on the ALU pipe.
//
// Each warp loads its 32 rows' bins coalesced (4 lanes per 64-byte row
// chunk), prefetches the next chunk into registers and transposes through a
// private shared buffer — warps never wait for each other inside a tile.
// Work is scheduled dynamically in items = (block of rows, word slice),
// ordered block-major, so CTAs working concurrently on the same row block
// share its bins through L2 (each row's bins leave HBM ~once); a CTA rebuilds
// its table only when its slice changes.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "hv_internal.cuh"

namespace hvb {

// table rows per feature: TB = 16 (B <= 16, the reference default) or 32
// (B <= 32: twice the table per word pair, so fewer pairs per lane fit)
constexpr int kChunk = 64;     // features per staged chunk

// Per feature and lane: 1 PRMT + NPR LDS.64 + 2*NW LOP3 (the previous version,
// one pair per lane, spent PRMT + LEA + LDS.64 + 4 LOP3 per pair: 3 ALU ops
// per bound word instead of 2.1; profiles/ncu_encode_r1_v5.txt shows it
// ALU-bound at 94 %).
struct TT6Params {
  const uint8_t* bins8;
  uint32_t ldb;
  uint64_t rows;
  uint32_t F, Fpad, D, W, B;  // Fpad: F rounded up to a multiple of 8 (zero table rows)
  const uint32_t* id;
  const uint32_t* val;
  const uint32_t* tie;
  uint32_t* out;
  uint32_t w0, wcount;  // output words [w0, w0 + wcount) of the W-word codebook rows
  uint32_t ldo;         // output row stride (words); word w0 + k goes to out[row * ldo + k]
  uint32_t slices;      // ceil(wcount / NW)
  uint32_t block_rows;  // rows per work item
  uint64_t blocks;      // ceil(rows / block_rows)
  unsigned int* counter;
  uint32_t perm;        // permutation binding: bound word = rotate(V_b, f) (encoding.cpp:273-279)
  // streamed input (host staging pipeline): rows [0, *ready) of bins8 have
  // landed; an item waits until its block's rows have; ~0 = aborted (rows
  // past the landed ones were never validated). nullptr = all resident.
  const unsigned long long* ready;
};

template <int NW>
struct Words {
  uint32_t v[NW];
};

// Harley–Seal over 2^K inputs of NW independent counters; s[k] has weight 2^k,
// the returned carries weight 2^K.
template <int K, int NW, class Load>
__device__ __forceinline__ Words<NW> hs_tree(uint32_t (&s)[6][NW], Load& ld) {
  Words<NW> h;
  if constexpr (K == 1) {
    const Words<NW> x = ld();
    const Words<NW> y = ld();
#pragma unroll
    for (int i = 0; i < NW; ++i) csa(h.v[i], s[0][i], s[0][i], x.v[i], y.v[i]);
  } else {
    const Words<NW> c1 = hs_tree<K - 1, NW>(s, ld);
    const Words<NW> c2 = hs_tree<K - 1, NW>(s, ld);
#pragma unroll
    for (int i = 0; i < NW; ++i) csa(h.v[i], s[K - 1][i], s[K - 1][i], c1.v[i], c2.v[i]);
  }
  return h;
}

// Majority by a biased counter. The planes (s[0..5], hi[0..NH-1]: K = 6 + NH
// bits, F < 2^K) start at b = 2^(K-1) - T, T = ceil(F / 2), so the count
// c + b never overflows K bits and
//     2c > F  <=>  c >= T + (F even)   2c == F  <=>  c == T (F even)
// c >= T is the top plane; c == T is the top plane with every lower plane
// zero. So bit = top for odd F, top & (any lower plane | tie) for even F:
// 4-6 LOP3 per word instead of a 2-op-per-plane compare against F / 2 with
// per-plane selects on the runtime F (round 1: ~50 ops per output word).
template <int NH>
__device__ __forceinline__ uint32_t majority_biased(const uint32_t (&pl)[6 + NH], bool odd, uint32_t tie) {
  constexpr int K = 6 + NH;
  uint32_t any = 0;
#pragma unroll
  for (int k = 0; k < K - 1; ++k) any |= pl[k];
  return pl[K - 1] & (odd ? 0xFFFFFFFFu : (any | tie));
}

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* a) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(a) : "memory");
  return v;
}

template <int NPR, int G, int NH, int MINB, bool PERM, int TB>
__global__ void __launch_bounds__(G * 32, MINB) encode_tt6_kernel(TT6Params p) {
  constexpr int NW = 2 * NPR;
  constexpr int kTBins = TB;
  constexpr uint32_t kFeatBytes = NPR * kTBins * 8;  // one feature's entries (all pairs)
  constexpr uint32_t kBinMask = TB == 16 ? 0x0F0F0F0Fu : 0x1F1F1F1Fu;  // b * 8 <= 248 still fits a byte
  extern __shared__ __align__(256) uint8_t sm6[];
  __shared__ unsigned int s_item;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  constexpr uint32_t nthreads = G * 32;
  const uint32_t tbytes = p.Fpad * kFeatBytes;  // multiple of 256 (Fpad % 8 == 0)
  uint32_t* Sw = reinterpret_cast<uint32_t*>(sm6 + tbytes) + warp * (16 * 32);  // [16 words][32 rows]
  const uint64_t items = static_cast<uint64_t>(p.slices) * p.blocks;
  const uint32_t nchunks = (p.Fpad + kChunk - 1) / kChunk;
  uint32_t cur_slice = 0xFFFFFFFFu;
  const uint32_t lr = lane >> 2, lq = lane & 3u;

  for (;;) {
    if (threadIdx.x == 0) {
      const unsigned int it = atomicAdd(p.counter, 1u);
      s_item = it;
      if (p.ready != nullptr && it < items) {
        // the copies that fill bins8 and then advance *ready run on a copy
        // engine, so waiting here cannot block them (no SM is needed)
        const uint64_t end = (it / p.slices + 1) * static_cast<uint64_t>(p.block_rows);
        const unsigned long long need = end < p.rows ? end : p.rows;
        unsigned long long v;
        while ((v = ld_acquire_u64(p.ready)) < need) __nanosleep(256);
        if (v == ~0ull) s_item = 0xFFFFFFFFu;  // the host aborted the call (bad bin): stop, output discarded
      }
    }
    __syncthreads();
    const uint64_t item = s_item;
    __syncthreads();
    if (item >= items) break;
    const uint32_t slice = static_cast<uint32_t>(item % p.slices);
    const uint64_t block = item / p.slices;
    const uint32_t wb = slice * NW;  // first local output word of the slice
    if (slice != cur_slice) {
      // entry (f, b): NW bound words (ID_f[w] ^ V_b[w], or rotate(V_b, f)[w]), w = w0+wb+j; zero for f >= F, b >= B, past the range
      for (uint32_t k = threadIdx.x; k < p.Fpad * kTBins; k += nthreads) {
        const uint32_t f = k / kTBins, b = k % kTBins;
        uint32_t e[NW];
#pragma unroll
        for (int j = 0; j < NW; ++j) {
          const uint32_t w = p.w0 + wb + j;
          if constexpr (PERM) {  // word w of V_b rotated by f (bits past D are masked at the output)
            e[j] = (wb + j < p.wcount && f < p.F && b < p.B)
                       ? get_bits_cyclic(p.val + static_cast<uint64_t>(b) * p.W, p.W, p.D,
                                         (w * 32u + p.D - (f % p.D)) % p.D)
                       : 0u;
          } else {
            e[j] = (wb + j < p.wcount && f < p.F && b < p.B)
                       ? __ldg(p.id + static_cast<uint64_t>(f) * p.W + w) ^ __ldg(p.val + static_cast<uint64_t>(b) * p.W + w)
                       : 0u;
          }
        }
#pragma unroll
        for (int t = 0; t < NPR; ++t) {
          *reinterpret_cast<uint2*>(sm6 + f * kFeatBytes + t * (kTBins * 8) + b * 8) = make_uint2(e[2 * t], e[2 * t + 1]);
        }
      }
      cur_slice = slice;
      __syncthreads();
    }
    const uint64_t r_begin = block * p.block_rows;
    const uint64_t r_end = min(p.rows, r_begin + p.block_rows);
    // counter bias b = 2^(K-1) - ceil(F / 2) as per-plane all-ones / zero masks
    const uint32_t bias = (1u << (5 + NH)) - ((p.F + 1) >> 1);
    const bool odd = p.F & 1u;
    for (uint64_t wrow0 = r_begin + 32ull * warp; wrow0 < r_end; wrow0 += 32ull * G) {
      uint32_t s[6][NW];
      uint32_t hi[NH][NW];
#pragma unroll
      for (int i = 0; i < NW; ++i) {
#pragma unroll
        for (int k = 0; k < 6; ++k) s[k][i] = 0u - ((bias >> k) & 1u);
#pragma unroll
        for (int k = 0; k < NH; ++k) hi[k][i] = 0u - ((bias >> (6 + k)) & 1u);
      }
      // coalesced loads: request i -> row 8i + lr, bytes 16*lq .. 16*lq+15 of the chunk
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
      for (int i = 0; i < 4; ++i) ld4[i] = __ldg(src[i]);  // rows past the block read row 0 (results not stored)
      // transpose into [w][r ^ 8*(w>>2)], bins scaled to table byte offsets (b*8).
      // Bins of features < F arrive validated (< B <= 16), so full chunks need no
      // nibble mask: the shift alone turns 4 bins into 4 table offsets (b * 8 < 128,
      // no carry between bytes). The last chunk holds the row padding [F, Fpad),
      // whose bytes the caller need not zero: masked to a nibble they index the
      // all-zero table rows of features >= F instead of running past the table.
      auto stage = [&](auto masked) {
        constexpr uint32_t m = decltype(masked)::value ? kBinMask : 0xFFFFFFFFu;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const uint32_t col = (8 * i + lr) ^ (lq << 3);
          Sw[(4 * lq + 0) * 32 + col] = (ld4[i].x & m) << 3;
          Sw[(4 * lq + 1) * 32 + col] = (ld4[i].y & m) << 3;
          Sw[(4 * lq + 2) * 32 + col] = (ld4[i].z & m) << 3;
          Sw[(4 * lq + 3) * 32 + col] = (ld4[i].w & m) << 3;
        }
      };
      if (nchunks == 1) stage(std::true_type{}); else stage(std::false_type{});
      __syncwarp();
      for (uint32_t ch = 0; ch < nchunks; ++ch) {
        const bool more = ch + 1 < nchunks;
        if (more) {
#pragma unroll
          for (int i = 0; i < 4; ++i) ld4[i] = __ldg(src[i] + (ch + 1) * (kChunk / 16));
        }
        const uint32_t tch = ch * (kChunk * kFeatBytes);  // 256-aligned chunk base (byte offset in sm6)
        int i = 0;
        uint32_t word = 0;
        auto ld = [&]() -> Words<NW> {
          // (indexing Sw directly keeps this an LDS; through an array of pointers it
          // compiled to generic LD.E plus a local-memory pointer table)
          if ((i & 3) == 0) word = Sw[(lane ^ ((static_cast<uint32_t>(i) >> 4 & 3u) << 3)) + (i >> 2) * 32];
          const uint32_t off = __byte_perm(word, tch, 0x7650 | (i & 3));
          const uint8_t* e = sm6 + off + i * kFeatBytes;
          Words<NW> v;
#pragma unroll
          for (int t = 0; t < NPR; ++t) {
            const uint2 x = *reinterpret_cast<const uint2*>(e + t * (kTBins * 8));
            v.v[2 * t] = x.x;
            v.v[2 * t + 1] = x.y;
          }
          ++i;
          return v;
        };
        const uint32_t nf = min(static_cast<uint32_t>(kChunk), p.Fpad - ch * kChunk);  // multiple of 8
        Words<NW> carry;  // weight 64, rippled into hi
        if (nf == kChunk) {
          carry = hs_tree<6, NW>(s, ld);
        } else {
          // 0..3 blocks of 16 and 0..1 block of 8 (< 64 features): carries of
          // weight 16 half-add into levels 4 and 5, a block of 8's carry into 3..5
#pragma unroll
          for (int j = 0; j < NW; ++j) carry.v[j] = 0;
          auto add16 = [&](const Words<NW>& c16) {
#pragma unroll
            for (int j = 0; j < NW; ++j) {
              const uint32_t c32 = s[4][j] & c16.v[j];
              s[4][j] ^= c16.v[j];
              const uint32_t c64 = s[5][j] & c32;
              s[5][j] ^= c32;
              carry.v[j] |= c64;  // at most one weight-64 carry per bit: the chunk adds < 64
            }
          };
          // two weight-16 carries enter level 4 through one carry-save adder
          auto add16x2 = [&](const Words<NW>& ca, const Words<NW>& cb) {
#pragma unroll
            for (int j = 0; j < NW; ++j) {
              uint32_t c32;
              csa(c32, s[4][j], s[4][j], ca.v[j], cb.v[j]);
              const uint32_t c64 = s[5][j] & c32;
              s[5][j] ^= c32;
              carry.v[j] |= c64;
            }
          };
          auto c8to16 = [&]() {  // a block of 8: its weight-8 carry half-adds into level 3
            const Words<NW> c8 = hs_tree<3, NW>(s, ld);
            Words<NW> c16;
#pragma unroll
            for (int j = 0; j < NW; ++j) {
              c16.v[j] = s[3][j] & c8.v[j];
              s[3][j] ^= c8.v[j];
            }
            return c16;
          };
          const uint32_t n16 = nf >> 4;
          const bool has8 = nf & 8u;
          if (n16 >= 2) {
            const Words<NW> ca = hs_tree<4, NW>(s, ld);
            add16x2(ca, hs_tree<4, NW>(s, ld));
          }
          if (n16 == 1 || n16 == 3) {
            const Words<NW> ca = hs_tree<4, NW>(s, ld);
            if (has8) {
              add16x2(ca, c8to16());
            } else {
              add16(ca);
            }
          } else if (has8) {
            add16(c8to16());
          }
        }
#pragma unroll
        for (int j = 0; j < NW; ++j) {
          uint32_t c = carry.v[j];
#pragma unroll
          for (int k = 0; k < NH - 1; ++k) {
            const uint32_t t = hi[k][j] & c;
            hi[k][j] ^= c;
            c = t;
          }
          hi[NH - 1][j] ^= c;  // the biased count stays below 2^K: no carry out of the top plane
        }
        if (more) {
          __syncwarp();  // every lane has read its words of this chunk
          if (ch + 2 == nchunks) stage(std::true_type{}); else stage(std::false_type{});
          __syncwarp();
        }
      }
      const uint64_t row = wrow0 + lane;
      if (row < r_end) {
        uint32_t* o = p.out + row * p.ldo;
#pragma unroll
        for (int j = 0; j < NW; ++j) {
          const uint32_t w = p.w0 + wb + j;
          if (wb + j < p.wcount) {
            uint32_t pl[6 + NH];
#pragma unroll
            for (int k = 0; k < 6; ++k) pl[k] = s[k][j];
#pragma unroll
            for (int k = 0; k < NH; ++k) pl[6 + k] = hi[k][j];
            o[wb + j] = majority_biased<NH>(pl, odd, __ldg(p.tie + w)) & valid_mask(w, p.D);
          }
        }
      }
      __syncwarp();  // the staging buffer is rewritten by the next tile
    }
  }
}

namespace {

template <int NPR, int G, int NH, int MINB, int TB>
void launch_tt6_inst(hv_context* ctx, cudaStream_t st, TT6Params p, size_t smem) {
  // separate instantiations: the permutation table build must not perturb the
  // ID-level kernel's code (it cost 1.5 % there as a runtime branch)
  auto kern = p.perm ? encode_tt6_kernel<NPR, G, NH, MINB, true, TB> : encode_tt6_kernel<NPR, G, NH, MINB, false, TB>;
  ck(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)),
     "cudaFuncSetAttribute");
  int per_sm = 0;
  ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, G * 32, smem), "occupancy");
  if (per_sm < 1) fail(HV_ERR_CUDA, "encode_tt6_kernel: configuration does not fit on an SM");
  const uint64_t items = static_cast<uint64_t>(p.slices) * p.blocks;
  const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(items, static_cast<uint64_t>(ctx->sm_count) * per_sm));
  ck(cudaMemsetAsync(p.counter, 0, sizeof(unsigned int), st), "counter reset");
  kern<<<grid, G * 32, smem, st>>>(p);
  launched("encode_tt6_kernel");
}

bool launch_v6(hv_context* ctx, cudaStream_t st, const uint8_t* bins8, uint32_t ldb, uint64_t rows, uint32_t F,
               const uint32_t* id, const uint32_t* val, uint32_t B, uint32_t D, uint32_t W, const uint32_t* tie,
               uint32_t* out, uint32_t w0, uint32_t wcount, uint32_t ldo, uint32_t* counter, bool perm,
               const unsigned long long* ready) {
  // zero-padded feature count: a multiple of 8 (the partial chunk runs blocks of
  // 16 and 8), unless padding to 16 completes a 64-feature chunk (the full-chunk
  // tree is cheaper per feature): CHB-MIT 342 -> 344 (was 352), UCI-HAR 561 -> 576
  const uint32_t F16 = (F + 15) / 16 * 16;
  const uint32_t Fpad = (F16 % kChunk == 0) ? F16 : (F + 7) / 8 * 8;
  // planes above the six HS levels: counts < 64 * 2^NH; instantiated NH in {3, 4, 6}
  int nh = 0;
  while ((64ull << nh) <= F) ++nh;
  nh = nh <= 3 ? 3 : nh <= 4 ? 4 : nh <= 6 ? 6 : -1;
  if (nh < 0) return false;
  const int tb = B <= 16 ? 16 : 32;
  const size_t pair_table = static_cast<size_t>(Fpad) * tb * 8;
  const size_t wstage = 16 * 32 * 4;
  // Shapes (word pairs per lane, warps per CTA, CTAs per SM), preferred first.
  // Round 2: 12 warps (three per scheduler) with 3 or 2 pairs beat 8 warps
  // with 4 or 2 pairs by 3.1-3.5 % at every benchmark shape (E 16.43 -> 15.86,
  // H 27.15 -> 26.30, I 30.24 -> 29.21, M 37.38 -> 36.14 ms per 1 M rows:
  // profiles/encode_shapes_r2.txt); 10 warps (3+3+2+2 per scheduler) and 16
  // (128 registers, spills) lose. Round 1: 4 or 3 pairs with 8 warps beat 2
  // pairs with 2 CTAs/SM by 7 %, 1 pair by 22 %.
  struct Shape { int npr, g, minb; };
  // (32 bins: pair tables are twice as large, so the same list picks fewer
  // pairs; only the {2,8,1} and {1,8,2} shapes are instantiated for it)
  const Shape shapes[] = {{3, 12, 1}, {2, 12, 1}, {4, 8, 1}, {3, 8, 1}, {2, 8, 1}, {1, 8, 2}};
  constexpr int kShapes = sizeof(shapes) / sizeof(shapes[0]);
  const size_t two = 113 * 1024, one = std::min<size_t>(ctx->smem_optin, 225 * 1024);
  int pick = -1;
  const char* env = getenv("HVB200_TT_SHAPE");  // tuning override "npr,g,minb"
  int enp = 0, eg = 0, emb = 0;
  const bool forced = env && sscanf(env, "%d,%d,%d", &enp, &eg, &emb) == 3;
  for (int i = 0; i < kShapes; ++i) {
    const Shape& s = shapes[i];
    const size_t need = s.npr * pair_table + s.g * wstage;
    const bool inst = (tb == 16 || s.npr <= 2) && (s.g == 8 || tb == 16);
    const bool fits = inst && need <= (s.minb == 2 ? two : one);
    if (forced ? (s.npr == enp && s.g == eg && s.minb == emb && fits) : (fits && pick < 0)) pick = i;
  }
  if (pick < 0) return false;
  const Shape s = shapes[pick];
  const size_t smem = s.npr * pair_table + s.g * wstage;
  const uint32_t slices = static_cast<uint32_t>((wcount + 2 * s.npr - 1) / (2 * s.npr));
  // 16k-row blocks (bins of a block stay in L2 while its slices run), smaller
  // when that would leave fewer than ~4 items per CTA (chunked host pipelines)
  // (a multiple of 32 rows per warp of the CTA, so every warp gets as many
  // 32-row groups: 16,512 = 43 x 384 for 12 warps)
  const uint32_t unit = 32u * static_cast<uint32_t>(s.g);
  uint32_t block_rows = (16384u + unit / 2) / unit * unit;
  const uint64_t want_items = 4ull * ctx->sm_count * s.minb;
  if (((rows + block_rows - 1) / block_rows) * slices < want_items) {
    const uint64_t br = (rows * slices + want_items - 1) / want_items;
    block_rows = static_cast<uint32_t>(std::max<uint64_t>(unit, (br + unit - 1) / unit * unit));
  }
  if (const char* br_env = getenv("HVB200_TT_BLOCK_ROWS")) {  // tuning override: a positive multiple of 32
    const long v = strtol(br_env, nullptr, 10);
    if (v >= 32 && v <= (1l << 30)) block_rows = static_cast<uint32_t>(v / 32 * 32);
  }
  TT6Params p{bins8, ldb, rows, F, Fpad, D, W, B, id, val, tie, out, w0, wcount, ldo, slices, block_rows,
              (rows + block_rows - 1) / block_rows, counter, perm ? 1u : 0u, ready};
#define HV_TT6(NPR, G, MB, N, TB)                                        \
  if (s.npr == NPR && s.g == G && s.minb == MB && nh == N && tb == TB) { \
    launch_tt6_inst<NPR, G, N, MB, TB>(ctx, st, p, smem);                \
    return true;                                                         \
  }
#define HV_TT6_NH(NPR, G, MB, TB) HV_TT6(NPR, G, MB, 3, TB) HV_TT6(NPR, G, MB, 4, TB) HV_TT6(NPR, G, MB, 6, TB)
  HV_TT6_NH(4, 8, 1, 16)
  HV_TT6_NH(3, 12, 1, 16)
  HV_TT6_NH(2, 12, 1, 16)
  HV_TT6_NH(3, 8, 1, 16)
  HV_TT6_NH(2, 8, 1, 16)
  HV_TT6_NH(1, 8, 2, 16)
  HV_TT6_NH(2, 8, 1, 32)
  HV_TT6_NH(1, 8, 2, 32)
#undef HV_TT6_NH
#undef HV_TT6
  return false;
}

}  // namespace

bool launch_tt(hv_context* ctx, cudaStream_t st, const uint8_t* bins8, uint32_t ldb, uint64_t rows, uint32_t F,
               const uint32_t* id, const uint32_t* val, uint32_t B, uint32_t D, uint32_t W, const uint32_t* tie,
               uint32_t* out, uint32_t w0, uint32_t wcount, uint32_t ldo, bool perm,
               const unsigned long long* ready) {
  if (B > 32u || F == 0 || rows == 0 || wcount == 0) return false;
  if (ldb % kChunk != 0 || (reinterpret_cast<uintptr_t>(bins8) & 15u)) return false;
  // one work counter per launch from the context's ring (concurrent launches on
  // the context's two streams must not share one)
  unsigned int* counter = ctx->d_counters + (ctx->next_counter++ % hv_context::kCounters);
  return launch_v6(ctx, st, bins8, ldb, rows, F, id, val, B, D, W, tie, out, w0, wcount, ldo, counter, perm, ready);
}

}  // namespace hvb
