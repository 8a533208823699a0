// hv_predict_tc.cu — the many-class Hamming scan (model.cpp:69-79, 96-104,
// 303-320) on the 5th-generation tensor cores, rows in TMEM.
//
//   popc(q ^ c) = |q| + |c| - 2 <q, c>
//
// <q, c> is a 0/1 GEMM, rows x D times D x classes, computed with
// tcgen05.mma kind::f8f6f4: every bit becomes the e4m3 byte 0x08 (= 2^-6) or
// 0, so each product is 2^-12 or 0 and the f32 accumulator holds
// <q, c> * 2^-12 exactly (integers below 2^24 times a power of two). kind::i8
// with 0/1 bytes measured 1.5-2.6x slower per instruction on this B200.
// A CTA owns a PAIR of 128-row tiles against one class tile of N <= 128
// classes, two accumulators in TMEM (2 x 128 columns). The K dimension is the
// hypervector's bits, 128 per MMA stage (4 packed words).
//
//   * classes (B operand): spread once per call by tc_arrange_classes_kernel
//     into the exact shared-memory image the UMMA descriptor reads (K-major,
//     no swizzle, 8 x 16-byte core matrices), one 16 KB image per (class tile,
//     4-word stage); the CTA fetches it with one cp.async.bulk per chunk (async proxy,
//     completion through the stage's mbarrier transaction count);
//   * rows (A operand): 4 loader warps keep kRing 32-word chunks of packed rows
//     in flight with 16-byte cp.async into a shared ring (8 lanes per row, so
//     a warp's copy touches 4 lines); 8 spreader warps (one thread per row)
//     turn 4 words at a time into 32 byte-columns and write them
//     straight into TMEM with tcgen05.st — the MMA reads A from TMEM, so no
//     generic-proxy shared store (and no per-chunk proxy fence, whose MEMBAR
//     dominated the shared-memory-staged kernel) sits on the critical path;
//   * a dedicated MMA warp (one thread) waits for the stage's rows (an
//     mbarrier the 8 spreader warps arrive on after tcgen05.st) and class
//     image, issues 2 x 4 UMMAs (K = 128 bits) and commits them to the stage's mbarrier,
//     which frees both the TMEM A stage and the B stage — no CTA-wide barrier
//     in the steady state;
//   * the epilogue reads the f32 dot products out of TMEM (tcgen05.ld 32x32b,
//     thread = row) and folds |q| + |c| - 2<q,c> into the (distance, class)
//     argmin key exactly like the other scans.
//
// The bit -> byte spread is "strided" (byte 4j + b of a word's 32-byte K slice
// holds bit 8b + j); rows and classes use the same order, which the dot
// product does not see. MMA stages are half chunks (128 K bytes, 4 stages).
#include <cstdint>
#include <cstdlib>

#include "hv_internal.cuh"
#include "hv_scan_tc.cuh"

namespace hvb {
namespace {

// Raw row chunks are 32 words (one 128-byte line of an aligned row): 8
// loader lanes cover a row, so a warp's cp.async touches 4 lines instead of 32.
constexpr uint32_t kWords = 32;
// MMA stages are 4 words (128 K bytes); 4 stages in flight keep the tensor
// pipe fed while the spreaders refill the oldest one
constexpr uint32_t kSubWords = 4, kSubBytes = 32 * kSubWords, kSubSbo = (kSubBytes / 16) * 128;
constexpr uint32_t kStages = 4;
constexpr uint32_t kRows = 2 * tc::kM;        // rows per CTA work item (two accumulators)
// raw row chunks in flight: 4 for the full scan, 3 for the split-K popcount
// variant, whose epilogue transpose needs the shared memory
template <bool PARTIAL>
constexpr int kRingOf = PARTIAL ? 3 : 4;
constexpr int kSpread = 256, kLoad = 128, kThreads = kSpread + kLoad + 64;  // + class-image warp + MMA warp
constexpr uint32_t kImgWarp = (kSpread + kLoad) / 32, kMmaWarp = kImgWarp + 1;
// words per raw row slot: 32 + the 16-byte alignment window of unaligned rows;
// the 144-byte stride also makes 8 consecutive rows' 16-byte reads conflict-free
constexpr uint32_t kWin = kWords + 4;
constexpr uint32_t kImg = tc::kN * kSubBytes;  // class image bytes per (class tile, half chunk)
// TMEM columns: accumulators [0, 128) and [128, 256); A stages at 256 + 32 * (2 * stage + tile)
constexpr uint32_t kTmemCols = 512, kAcol = 256, kAcols = kSubBytes / 4;

template <bool PARTIAL>
struct __align__(1024) Smem {
  static constexpr int kRing = kRingOf<PARTIAL>;
  uint8_t b[kStages][kImg];
  uint32_t raw[kRing][kRows][kWin];
  uint32_t xpose[PARTIAL ? kSpread / 32 : 1][32][33];  // split-K epilogue: (row, class) -> (class, row) per warp
  unsigned long long mma_done[kStages], a_full[kStages], b_full[kStages], acc_empty;
  unsigned long long raw_full[kRing], raw_empty[kRing];
  uint32_t tmem;
};
template <bool PARTIAL>
constexpr size_t kSmemBytes = sizeof(Smem<PARTIAL>) + 1024;

// bit -> e4m3 byte: 0x08 (= 2^-6) or 0; byte b of spread word j holds bit 8b + j
template <uint32_t J>
__device__ __forceinline__ uint32_t spread(uint32_t x) {
  return (J <= 3 ? (x << (3 - J)) : (x >> (J - 3))) & 0x08080808u;
}

// kind::f8f6f4, A e4m3 from TMEM, B e4m3 from shared memory, D f32 in TMEM
__device__ __forceinline__ void mma_f8_ts(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
      "r"(a), "l"(bdesc), "r"(idesc), "r"(acc));
}

// 32 columns of this warp's 32 TMEM lanes from v[0..31] (thread = lane)
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
      "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]),
      "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]),
      "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
        "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t mbar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(mbar)
               : "memory");
}

// classes -> UMMA B images: img[ct * nsub + q] holds classes ct*128 .. +127,
// the K bytes of half chunk q (words 4q .. 4q+3), K-major no-swizzle core
// matrices: K byte k of class c at (c/8)*kSubSbo + (k/16)*128 + (c%8)*16 + k%16.
// cpop (optional): the first blocks also write each class's popcount (warp per class).
__global__ void tc_arrange_classes_kernel(const uint32_t* __restrict__ cv, uint32_t C, uint32_t W, uint32_t nct,
                                          uint32_t nsub, uint8_t* __restrict__ img, uint32_t* __restrict__ cpop) {
  if (cpop != nullptr) {
    const uint32_t c = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5), lane = threadIdx.x & 31u;
    if (c < C) {
      uint32_t a = 0;
      for (uint32_t w = lane; w < W; w += 32) a += __popc(cv[static_cast<uint64_t>(c) * W + w]);
      a = __reduce_add_sync(0xFFFFFFFFu, a);
      if (lane == 0) cpop[c] = a;
    }
  }
  const uint64_t total = static_cast<uint64_t>(nct) * nsub * tc::kN * kSubWords;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t kw = static_cast<uint32_t>(i % kSubWords);
    const uint32_t c = static_cast<uint32_t>((i / kSubWords) % tc::kN);
    const uint64_t tk = i / (kSubWords * tc::kN);  // ct * nsub + q
    const uint32_t q = static_cast<uint32_t>(tk % nsub), ct = static_cast<uint32_t>(tk / nsub);
    const uint32_t cls = ct * tc::kN + c, w = q * kSubWords + kw;
    const uint32_t x = (cls < C && w < W) ? cv[static_cast<uint64_t>(cls) * W + w] : 0u;
    uint4* dst = reinterpret_cast<uint4*>(img + tk * kImg + (c >> 3) * kSubSbo + (c & 7u) * 16 + 2 * kw * 128);
    dst[0] = make_uint4(spread<0>(x), spread<1>(x), spread<2>(x), spread<3>(x));
    dst[8] = make_uint4(spread<4>(x), spread<5>(x), spread<6>(x), spread<7>(x));  // +128 bytes
  }
}

// One CTA work item: a pair of row tiles x one class tile x one K range (a
// split of the 32-word chunks; ks = 1 covers the whole hypervector).
struct Item {
  uint32_t ct, k0, k1, q0, q1;
  uint64_t row0;
};
__device__ __forceinline__ Item item_of(uint64_t it, uint32_t nct, uint32_t ks, uint32_t nchunks, uint32_t nsub) {
  Item m;
  const uint32_t kx = static_cast<uint32_t>(it % ks);
  const uint64_t rest = it / ks;
  m.ct = static_cast<uint32_t>(rest % nct);
  m.row0 = (rest / nct) * kRows;
  m.k0 = static_cast<uint32_t>(static_cast<uint64_t>(nchunks) * kx / ks);
  m.k1 = static_cast<uint32_t>(static_cast<uint64_t>(nchunks) * (kx + 1) / ks);
  m.q0 = m.k0 * (kWords / kSubWords);
  m.q1 = min(m.k1 * (kWords / kSubWords), nsub);
  return m;
}

// ALIGNED: every row starts 16-byte aligned (W % 4 == 0); otherwise each raw
// slot holds the 16-byte-aligned 144-byte window around the row's chunk and
// the spreader picks its words at the row's word offset.
template <bool ALIGNED, bool PARTIAL>
__global__ void __launch_bounds__(kThreads, 1)
    predict_tc_kernel(const uint8_t* __restrict__ img, uint32_t C, uint32_t N, uint32_t D, uint32_t W,
                      const uint32_t* __restrict__ enc, uint64_t rows, const uint32_t* __restrict__ cpop,
                      unsigned long long* __restrict__ best, double* __restrict__ dist, uint32_t* __restrict__ pops,
                      uint32_t ks) {
  extern __shared__ uint8_t tc_raw[];
  using SmemT = Smem<PARTIAL>;
  constexpr int kRing = SmemT::kRing;
  SmemT& s = *reinterpret_cast<SmemT*>((reinterpret_cast<uintptr_t>(tc_raw) + 1023) & ~uintptr_t(1023));
  if (!PARTIAL) ks = 1;
  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31u;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc::smem_u32(&s.tmem)),
                 "n"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (uint32_t st = 0; st < kStages; ++st) {
      tc::mbar_init(tc::smem_u32(&s.mma_done[st]), 1);
      tc::mbar_init(tc::smem_u32(&s.b_full[st]), 1);
      tc::mbar_init(tc::smem_u32(&s.a_full[st]), kSpread / 32);
    }
    tc::mbar_init(tc::smem_u32(&s.acc_empty), kSpread / 32);
    for (int r = 0; r < kRing; ++r) {
      tc::mbar_init(tc::smem_u32(&s.raw_full[r]), kLoad);
      tc::mbar_init(tc::smem_u32(&s.raw_empty[r]), kSpread / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = s.tmem;
  const uint32_t nct = (C + tc::kN - 1) / tc::kN;
  const uint64_t npairs = (rows + kRows - 1) / kRows;
  const uint32_t nchunks = (W + kWords - 1) / kWords, nsub = (W + kSubWords - 1) / kSubWords;
  // best == nullptr: popcounts only, split-K over ks items per tile; each item
  // ADDS its partial |q| - 2<q, c> (+ |c| for the first split) into pops
  // (mod 2^32, zeroed by the caller)
  const uint64_t items = npairs * nct * ks;
  if (warp == kMmaWarp) {
    // ---- MMA issue: one thread; per stage 2 x 4 UMMAs (A = the stage's TMEM rows, B = its class image)
    if (lane == 0) {
      // D f32, A and B e4m3, both K-major, N, M = 128
      const uint32_t idesc = (1u << 4) | ((N >> 3) << 17) | ((static_cast<uint32_t>(tc::kM) >> 4) << 24);
      uint32_t gch = 0, a_phase = 0, b_phase = 0, pair = 0;
      for (uint64_t it = blockIdx.x; it < items; it += gridDim.x, ++pair) {
        const Item m = item_of(it, nct, ks, nchunks, nsub);
        if (pair > 0) {  // the previous pair's epilogue has read the accumulators
          tc::mbar_wait(tc::smem_u32(&s.acc_empty), (pair - 1) & 1u);
        }
        for (uint32_t q = m.q0; q < m.q1; ++q, ++gch) {
          const uint32_t st = gch % kStages;
          tc::mbar_wait(tc::smem_u32(&s.a_full[st]), (a_phase >> st) & 1u);
          a_phase ^= 1u << st;
          tc::mbar_wait(tc::smem_u32(&s.b_full[st]), (b_phase >> st) & 1u);
          b_phase ^= 1u << st;
          asm volatile("tcgen05.fence::after_thread_sync;");
          const uint32_t b0 = tc::smem_u32(s.b[st]);
#pragma unroll
          for (uint32_t j = 0; j < kSubWords; ++j) {  // K = 32 bytes per UMMA: 8 A columns, 256 B of image
            const uint64_t bd = tc::make_desc(b0 + 256 * j, 128, kSubSbo);
            const uint32_t acc = (q != m.q0 || j != 0) ? 1u : 0u;
            mma_f8_ts(tmem, tmem + kAcol + kAcols * (2 * st + 0) + 8 * j, bd, idesc, acc);
            mma_f8_ts(tmem + tc::kN, tmem + kAcol + kAcols * (2 * st + 1) + 8 * j, bd, idesc, acc);
          }
          tc::commit(tc::smem_u32(&s.mma_done[st]));
        }
      }
    }
  } else if (warp == kImgWarp) {
    // ---- class images: one cp.async.bulk per chunk into B stage gch & 1, once its last MMAs are done
    if (lane == 0) {
      uint32_t gch = 0, mma_phase = 0, pending = 0;
      for (uint64_t it = blockIdx.x; it < items; it += gridDim.x) {
        const Item m = item_of(it, nct, ks, nchunks, nsub);
        const uint8_t* bimg = img + static_cast<uint64_t>(m.ct) * nsub * kImg;
        for (uint32_t q = m.q0; q < m.q1; ++q, ++gch) {
          const uint32_t st = gch % kStages;
          if ((pending >> st) & 1u) {
            tc::mbar_wait(tc::smem_u32(&s.mma_done[st]), (mma_phase >> st) & 1u);
            mma_phase ^= 1u << st;
          }
          pending |= 1u << st;
          bulk_g2s(tc::smem_u32(s.b[st]), bimg + static_cast<uint64_t>(q) * kImg, N * kSubBytes,
                   tc::smem_u32(&s.b_full[st]));
        }
      }
    }
  } else if (warp >= kSpread / 32) {
    // ---- row loaders: lane group t >> 3 takes rows (t >> 3) + 16 i, lane t & 7 the row's 16-byte piece
    const uint32_t t = tid - kSpread, pc = t & 7u, rg = t >> 3;
    uint32_t gch = 0;
    for (uint64_t it = blockIdx.x; it < items; it += gridDim.x) {
      const Item m = item_of(it, nct, ks, nchunks, nsub);
      const uint64_t row0 = m.row0;
      for (uint32_t kc = m.k0; kc < m.k1; ++kc, ++gch) {
        const uint32_t r = gch % kRing, ph = (gch / kRing) & 1u;
        tc::mbar_wait(tc::smem_u32(&s.raw_empty[r]), ph ^ 1u);
        const uint32_t w = kc * kWords;
#pragma unroll 4
        for (uint32_t i = 0; i < kRows / 16; ++i) {
          const uint32_t pr = rg + 16 * i;
          const uint64_t row = row0 + pr;
          const bool ok = row < rows;
          const uint32_t* src = enc + (ok ? row : 0) * W;
          const uint32_t dst = tc::smem_u32(&s.raw[r][pr][0]);
          if (ALIGNED) {
            const bool in = ok && w + 4 * pc < W;
            tc::cp_async16(dst + 16 * pc, src + (in ? w + 4 * pc : 0), in ? 16u : 0u);
          } else {
            // 144-byte window from the 16-byte boundary at or below word w of the row,
            // clamped to the row's end (bytes past it are zero-filled, never read)
            const uintptr_t a16 = reinterpret_cast<uintptr_t>(src + w) & ~uintptr_t(15);
            const uintptr_t end = reinterpret_cast<uintptr_t>(src + W);
#pragma unroll
            for (uint32_t q = 0; q < 2; ++q) {
              const uint32_t piece = pc + 8 * q;
              if (piece < kWin / 4) {
                const uintptr_t p = a16 + 16 * piece;
                const uint32_t n =
                    (!ok || p >= end) ? 0u : (end - p >= 16 ? 16u : static_cast<uint32_t>(end - p));
                tc::cp_async16(dst + 16 * piece, n ? reinterpret_cast<const void*>(p) : src, n);
              }
            }
          }
        }
        tc::cp_async_arrive(tc::smem_u32(&s.raw_full[r]));
      }
    }
  } else {
    // ---- spreaders: warp w owns TMEM lanes 32(w%4).. of tile w/4; thread = row
    const uint32_t tile = warp >> 2, lrow = ((warp & 3u) << 5) | lane, prow = tile * tc::kM + lrow;
    const uint32_t lane_base = (warp & 3u) << 21;  // (32 * (w % 4)) << 16
    uint32_t mma_phase = 0, pending = 0;
    uint32_t gch = 0, gsub = 0;
    for (uint64_t it = blockIdx.x; it < items; it += gridDim.x) {
      const Item m = item_of(it, nct, ks, nchunks, nsub);
      const uint32_t c0 = m.ct * tc::kN;
      const uint64_t row0 = m.row0;
      const uint64_t row = row0 + prow;
      uint32_t mis = 0;
      if (!ALIGNED) mis = static_cast<uint32_t>((reinterpret_cast<uintptr_t>(enc + (row < rows ? row : 0) * W) >> 2) & 3u);
      uint32_t rowpop = 0;
      for (uint32_t kc = m.k0; kc < m.k1; ++kc, ++gch) {
        const uint32_t r = gch % kRing, ph = (gch / kRing) & 1u;
        tc::mbar_wait(tc::smem_u32(&s.raw_full[r]), ph);
        const uint32_t base = tc::smem_u32(&s.raw[r][prow][0]);
        const uint32_t qend = min(kWords / kSubWords, nsub - kc * (kWords / kSubWords));
#pragma unroll 1
        for (uint32_t q = 0; q < qend; ++q, ++gsub) {  // words 4q..4q+3 of the chunk -> stage gsub % kStages
          uint32_t x[4];
          if (ALIGNED) {
            const uint4 u = tc::lds128(base + 16 * q);
            x[0] = u.x, x[1] = u.y, x[2] = u.z, x[3] = u.w;
          } else {
            const uint4 u = tc::lds128(base + 16 * q), v = tc::lds128(base + 16 * q + 16);
            const uint32_t win[8] = {u.x, u.y, u.z, u.w, v.x, v.y, v.z, v.w};
#pragma unroll
            for (uint32_t i = 0; i < 4; ++i) {
              x[i] = mis == 0 ? win[i] : mis == 1 ? win[i + 1] : mis == 2 ? win[i + 2] : win[i + 3];
            }
          }
          if (q + 1 == qend) {
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(tc::smem_u32(&s.raw_empty[r]));  // release orders the reads above
          }
          rowpop += __popc(x[0]) + __popc(x[1]) + __popc(x[2]) + __popc(x[3]);
          const uint32_t st = gsub % kStages;
          if ((pending >> st) & 1u) {  // the MMAs that last read this A stage are done
            tc::mbar_wait(tc::smem_u32(&s.mma_done[st]), (mma_phase >> st) & 1u);
            mma_phase ^= 1u << st;
          }
          pending |= 1u << st;
          uint32_t v[32];
#pragma unroll
          for (uint32_t i = 0; i < 4; ++i) {
            const uint32_t xi = x[i];
            v[8 * i + 0] = spread<0>(xi), v[8 * i + 1] = spread<1>(xi), v[8 * i + 2] = spread<2>(xi);
            v[8 * i + 3] = spread<3>(xi), v[8 * i + 4] = spread<4>(xi), v[8 * i + 5] = spread<5>(xi);
            v[8 * i + 6] = spread<6>(xi), v[8 * i + 7] = spread<7>(xi);
          }
          tmem_st32(tmem + lane_base + kAcol + kAcols * (2 * st + tile), v);
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
          asm volatile("tcgen05.fence::before_thread_sync;");
          __syncwarp();
          if (lane == 0) tc::mbar_arrive(tc::smem_u32(&s.a_full[st]));
        }
      }
      // every MMA of the pair has landed in TMEM
      for (uint32_t st = 0; st < kStages; ++st) {
        if ((pending >> st) & 1u) {
          tc::mbar_wait(tc::smem_u32(&s.mma_done[st]), (mma_phase >> st) & 1u);
          mma_phase ^= 1u << st;
        }
      }
      pending = 0;
      asm volatile("tcgen05.fence::after_thread_sync;");
      // epilogue: thread = row of its tile; accumulator columns 128 * tile ..
      const bool eok = row < rows;
      unsigned long long key = ~0ull;
#pragma unroll 1
      for (uint32_t cb = 0; cb < tc::kN / 32; ++cb) {
        if (32 * cb >= N) break;  // warp-uniform
        uint32_t v[32];
        tmem_ld32(tmem + lane_base + tc::kN * tile + 32 * cb, v);
        if (PARTIAL) {
          // partial (split-K) popcounts |q|_k - 2<q, c>_k (+ |c| once), mod 2^32,
          // transposed through shared memory so each warp-wide atomic covers 32
          // consecutive classes of one row
          uint32_t(&xp)[32][33] = s.xpose[warp];
#pragma unroll
          for (uint32_t i = 0; i < 32; ++i) {
            const uint32_t c = c0 + 32 * cb + i;
            const uint32_t dot = static_cast<uint32_t>(__uint_as_float(v[i]) * 4096.0f);
            xp[lane][i] = rowpop - 2u * dot + ((m.k0 == 0 && c < C) ? cpop[c] : 0u);
          }
          __syncwarp();
          const uint32_t c = c0 + 32 * cb + lane;
          const uint64_t wrow0 = row0 + tile * tc::kM + ((warp & 3u) << 5);
#pragma unroll 4
          for (uint32_t j = 0; j < 32; ++j) {
            if (c < C && wrow0 + j < rows) atomicAdd(pops + (wrow0 + j) * C + c, xp[j][lane]);
          }
          __syncwarp();
        } else if (eok) {
#pragma unroll
          for (uint32_t i = 0; i < 32; ++i) {
            const uint32_t c = c0 + 32 * cb + i;
            if (c < C) {
              // <q, c> * 2^-12, exact in f32 (D < 2^24)
              const uint32_t dot = static_cast<uint32_t>(__uint_as_float(v[i]) * 4096.0f);
              const uint32_t ham = rowpop + cpop[c] - 2u * dot;
              const unsigned long long k = (static_cast<unsigned long long>(ham) << 32) | c;
              key = k < key ? k : key;
              if (pops) pops[row * C + c] = ham;
              if (dist) dist[row * C + c] = static_cast<double>(ham) / static_cast<double>(D);
            }
          }
        }
      }
      if (eok && !PARTIAL) atomicMin(best + row, key);
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(tc::smem_u32(&s.acc_empty));  // accumulators free for the next pair
    }
  }
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kTmemCols));
}

}  // namespace

namespace {
// arrange the class images into img (nct * nsub * kImg bytes) and run the scan
// cpop_out: compute the class popcounts into it (cpop then points there)
void tc_scan(hv_context* ctx, cudaStream_t st, const uint32_t* cv, size_t C, size_t D, const uint32_t* enc,
             size_t rows, const uint32_t* cpop, unsigned long long* best, double* dist, uint32_t* pops, uint8_t* img,
             uint32_t ks, uint32_t* cpop_out = nullptr) {
  const size_t W = words_per_row(D);
  const uint32_t nct = static_cast<uint32_t>((C + tc::kN - 1) / tc::kN);
  const uint32_t nsub = static_cast<uint32_t>((W + kSubWords - 1) / kSubWords);
  // N: classes per UMMA, a multiple of 16 covering one class tile
  const uint32_t N = C >= tc::kN ? tc::kN : static_cast<uint32_t>((C + 15) / 16 * 16);
  const uint64_t work = static_cast<uint64_t>(nct) * nsub * tc::kN * kSubWords;
  const unsigned ag = std::max(grid_for(work, 256, ctx->sm_count * 8), static_cast<unsigned>((C + 7) / 8));
  tc_arrange_classes_kernel<<<ag, 256, 0, st>>>(cv, static_cast<uint32_t>(C), static_cast<uint32_t>(W), nct, nsub,
                                                 img, cpop_out);
  launched("tc_arrange_classes_kernel");
  if (cpop_out) cpop = cpop_out;
  const bool aligned = W % 4 == 0;
  const bool partial = best == nullptr;
  auto kern = partial ? (aligned ? predict_tc_kernel<true, true> : predict_tc_kernel<false, true>)
                      : (aligned ? predict_tc_kernel<true, false> : predict_tc_kernel<false, false>);
  const size_t smem = partial ? kSmemBytes<true> : kSmemBytes<false>;
  static bool attr_set[4] = {false, false, false, false};  // per process; the attribute is per function
  if (!attr_set[2 * partial + aligned]) {
    ck(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)),
       "cudaFuncSetAttribute");
    attr_set[2 * partial + aligned] = true;
  }
  const uint64_t items = ((rows + kRows - 1) / kRows) * nct * ks;
  const unsigned g = static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>(items, ctx->sm_count)));
  kern<<<g, kThreads, smem, st>>>(img, static_cast<uint32_t>(C), N, static_cast<uint32_t>(D),
                                        static_cast<uint32_t>(W), enc, rows, cpop, best, dist, pops, ks);
  launched("predict_tc_kernel");
}
}  // namespace

size_t tc_image_bytes(size_t C, size_t D) {
  const size_t W = words_per_row(D);
  return ((C + tc::kN - 1) / tc::kN) * ((W + kSubWords - 1) / kSubWords) * kImg;
}

bool tc_usable(const uint32_t* enc, size_t D) {
  return (reinterpret_cast<uintptr_t>(enc) & 15u) == 0 && D < (size_t(1) << 24);
}

bool predict_tc_launch(hv_context* ctx, cudaStream_t st, const uint32_t* cv, size_t C, size_t D, const uint32_t* enc,
                       size_t rows, const uint32_t* cpop, unsigned long long* best, double* dist, uint32_t* pops) {
  if (!tc_usable(enc, D)) return false;  // 16-byte copy windows; f32-exact dot products
  DevBuf<uint8_t> img(tc_image_bytes(C, D), st);
  tc_scan(ctx, st, cv, C, D, enc, rows, cpop, best, dist, pops, img.ptr, 1);
  return true;
}

void popc_tc_split(hv_context* ctx, cudaStream_t st, const uint32_t* cv, size_t C, size_t D, const uint32_t* enc,
                   size_t rows, uint32_t* cpop, uint32_t* pops, uint8_t* img) {
  const size_t W = words_per_row(D);
  const uint64_t base = ((rows + kRows - 1) / kRows) * ((C + tc::kN - 1) / tc::kN);
  const uint64_t nchunks = (W + kWords - 1) / kWords;
  const uint32_t ks = static_cast<uint32_t>(
      std::max<uint64_t>(1, std::min<uint64_t>(nchunks, (ctx->sm_count + base - 1) / base)));
  tc_scan(ctx, st, cv, C, D, enc, rows, nullptr, nullptr, nullptr, pops, img, ks, cpop);
}

}  // namespace hvb
