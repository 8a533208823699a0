// hv_encode_tc.cu — the ID-level encode (reference encoding.cpp:266-272) as a
// sparse FP4 GEMM on the 5th-generation tensor cores.
//
// counts[r][d] = sum_f bit_d(ID_f ^ V_{bin(r,f)}) = sum_k A[r][k] * T[k][d],
// k = 16 f + b: A is the one-hot bins of row r (F ones in 16 F columns), T the
// bound table (T[16 f + b][d] = bit d of ID_f ^ V_b, 0 or 1). The counts are
// exact in the fp32 accumulator (<= F), and the output bit is the reference's
// majority with tiebreak: 2 c > F, or 2 c == F and the tiebreak bit.
//
// A one-hot group of 8 logical K elements holds at most one 1, so A is
// "pair-wise 4:8" structured-sparse, the sparsity `tcgen05.mma.sp` takes for
// FP4: each group of 8 keeps 2 of its 4 element pairs (a 4-bit metadata nibble:
// low 2 bits = the pair of compressed elements 0-1, high 2 bits = the pair of
// elements 2-3), so a K = 128 (8 features) step of one row is 32 bytes of
// compressed e2m1 values plus 64 bits of metadata. Both are generated here from
// the row's 8 bin bytes with one 16-entry table lookup per feature; the
// metadata goes to TMEM (lane = row, one 32-bit column per 64 logical K), the
// values to shared memory in the UMMA's K-major no-swizzle layout. The bound
// table is built once per call as the exact shared-memory image of every
// (256-column N tile, K step) pair (16 KB each), streamed by one bulk copy per
// step. Scale factors (block16, ue4m3) are all 1.0: whole TMEM columns filled
// with 0x38 bytes. Measured on this B200 (scripts/probe_tc_fp4.cu): the sparse
// UMMA (M = 128, N = 256, K = 128) issues every 160 cycles = 14.2 PFLOP/s
// dense-equivalent; scripts/probe_tc_sparse_encode.cu checks the formats.
//
// CTA (one per SM, persistent over 128-row M tiles): warps 0-3 (thread = row)
// write the tile's compressed A images for every K step to an L2 scratch and
// its metadata to TMEM, once per tile, and run the epilogue; warp 4 streams
// (A image, bound-table image) pairs into as many shared-memory stages as fit
// with bulk copies; warp 5 issues one UMMA per K step into one of two TMEM
// accumulators (N = 192 while the tile's metadata fits beside them, else 128),
// so the epilogue of one N tile overlaps the next tile's MMAs.
//
// STATUS: a correct prototype, opt-in (HVB200_ENCODE_TC=1), bit-exact against
// the table encoder on every shape tested (tests/test_gpu_encode_tc.py), but
// SLOWER than it: 23.8 vs 15.9 ms per 1 M CHB-MIT rows (19.8 with no bulk
// copies and no epilogue). The probe's UMMA rates are exactly the operand
// bytes over 128 B/clk of shared-memory read: N = 128 / 192 / 256 read 4 KB of
// A + N x 64 B of B = 12 / 16 / 20 KB in 96 / 128 / 160 cycles. So the sparse
// FP4 UMMA at these shapes is shared-memory bound, not tensor bound, and with
// a fresh 16 KB stage per UMMA the bulk-copy writes double that traffic:
// 256 cycles per UMMA = 16.2 ms per 1 M rows, the ALU encoder's time, before
// any other loss. One mbarrier wait per two stages (28.2 ms) and relaxed
// waits (23.8) did not help. Only halving the staged bytes per FLOP can beat
// the ALU path: cta_group::2 (M = 256, B split across the SM pair: 12 KB read
// + 12 KB written per SM per 128 x 256 block, ~9 ms floor). DESIGN.md §8.
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "hv_internal.cuh"

namespace hvb {
namespace {

constexpr int kTM = 128;
constexpr uint32_t kAStage = kTM * 32;
constexpr uint32_t kTmemCols = 512;
// TMEM columns: two accumulators of TN, then 16 + 16 scale-factor columns, then
// 2 metadata columns per K step of the tile
template <int TN>
struct TcCfg {
  static constexpr uint32_t kBStage = TN * 64;
  // as many stages as shared memory holds: an UMMA's completion takes ~1.8 k
  // cycles after issue and a stage refill ~1 k (L2), so the ring must hold
  // that many cycles of MMAs for the tensor pipe to stay busy
  static constexpr int kStages = (225 * 1024) / (kTM * 32 + TN * 64);
  static constexpr uint32_t kColSfa = 2 * TN, kColSfb = 2 * TN + 16, kColMeta = 2 * TN + 32;
  static constexpr uint32_t kMaxKsteps = (kTmemCols - kColMeta) / 2;
};
constexpr int kThreads = 192;

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (static_cast<uint64_t>((saddr & 0x3FFFFu) >> 4)) | (static_cast<uint64_t>(lbo >> 4) << 16) |
         (static_cast<uint64_t>(sbo >> 4) << 32) | (1ull << 46);
}

__device__ __forceinline__ void mbar_init(uint32_t m, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(m), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint32_t m) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(m) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t m, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}\n" ::"r"(m),
      "r"(parity)
      : "memory");
}

// Bound-table image: for N tile nt and K step ks, TN rows (d) x 64 bytes
// (128 logical k = 8 features x 16 bins, e2m1 1.0 = nibble 0x2, element 2i in
// the low nibble), byte (n, c) at (n/8)*512 + (c/16)*128 + (n%8)*16 + c%16.
// One thread per (image, n, 16-byte chunk c/16).
template <int TN>
__global__ void tc_table_kernel(const uint32_t* __restrict__ id, const uint32_t* __restrict__ val, uint32_t F,
                                uint32_t B, uint32_t D, uint32_t W, uint32_t ksteps, uint32_t ntiles,
                                uint4* __restrict__ img) {
  constexpr int kTN = TN;
  const uint64_t total = static_cast<uint64_t>(ntiles) * ksteps * kTN * 4;
  for (uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t q = static_cast<uint32_t>(t & 3u);  // 16-byte chunk = 32 logical k = 2 features
    const uint32_t n = static_cast<uint32_t>((t >> 2) % kTN);
    const uint64_t im = (t >> 2) / kTN;
    const uint32_t ks = static_cast<uint32_t>(im % ksteps), nt = static_cast<uint32_t>(im / ksteps);
    const uint32_t d = nt * kTN + n;
    uint32_t w4[4] = {0u, 0u, 0u, 0u};
    if (d < D) {
      const uint32_t wd = d >> 5, bit = d & 31u;
#pragma unroll
      for (uint32_t h = 0; h < 2; ++h) {
        const uint32_t f = ks * 8u + q * 2u + h;
        if (f >= F) continue;
        const uint32_t idb = (__ldg(id + static_cast<uint64_t>(f) * W + wd) >> bit) & 1u;
        for (uint32_t b = 0; b < B && b < 16u; ++b) {
          const uint32_t tb = idb ^ ((__ldg(val + static_cast<uint64_t>(b) * W + wd) >> bit) & 1u);
          if (tb) {
            const uint32_t kk = h * 16u + b;          // logical k within the chunk (0..31)
            w4[kk >> 3] |= 0x2u << (4u * (kk & 7u));  // byte kk/2, low nibble for even kk
          }
        }
      }
    }
    const uint64_t off = im * (TcCfg<TN>::kBStage / 16) + (n / 8) * 32 + q * 8 + (n % 8);  // in uint4 units
    img[off] = make_uint4(w4[0], w4[1], w4[2], w4[3]);
  }
}

// Per bin b: the compressed bytes of the feature's two groups of 8 (bytes
// 2h, 2h+1 for group h: elements 0-1 = pair idx0, 2-3 = pair idx1) and the
// two metadata nibbles (group h at bits 4h..4h+3).
struct BinCode {
  uint32_t abytes;
  uint32_t meta;
};
__device__ __forceinline__ BinCode bin_code(uint32_t b) {
  const uint32_t h = b >> 3, p = (b & 7u) >> 1, e = b & 1u;
  const uint32_t v = e ? 0x20u : 0x02u;
  // group h keeps (idx0, idx1) = (0, 1) with the one in element pair 0, or (0, p) with it in pair p
  const uint32_t byte = 2u * h + (p == 0 ? 0u : 1u);
  const uint32_t nib_h = p == 0 ? (1u << 2) : (p << 2);  // idx0 = 0
  const uint32_t nib_o = 1u << 2;                         // the other group: (0, 1), zeros
  BinCode c;
  c.abytes = v << (8u * byte);
  c.meta = h == 0 ? (nib_h | (nib_o << 4)) : (nib_o | (nib_h << 4));
  return c;
}

struct TcParams {
  const uint8_t* bins8;
  uint32_t ldb;
  uint64_t rows;
  uint32_t F, D, W, ksteps, ntiles;
  const uint4* img;     // bound-table images [ntiles][ksteps][16 KB]
  uint4* scratch;       // per CTA: [ksteps][4 KB] compressed A images of its current M tile
  const uint32_t* tie;
  uint32_t* out;
  uint32_t ldo;
  uint32_t ablate;  // timing experiments only (HVB200_TC_ABLATE): 1 no copies, 4 no epilogue
  unsigned long long* prof;  // HVB200_TC_PROF=1: CTA 0's MMA thread cycles [total, full waits, acc waits, a_ready waits, issue]
};

// Per M tile (128 rows): warps 0-3 (thread = row) write the tile's compressed
// A images for every K step to this CTA's L2 scratch and its metadata for
// every K step to TMEM (columns kColMeta + 2 ks), once; then, per 256-column
// N tile, warp 4 streams (A image, bound-table image) pairs into kStages
// shared-memory stages with bulk copies (no generic-proxy shared stores on the
// pipeline, so no per-stage proxy fence), warp 5 issues one UMMA per K step,
// and warps 0-3 turn the accumulator into majority bits.
template <int TN>
__global__ void __launch_bounds__(kThreads, 1) encode_tc_kernel(TcParams p) {
  using Cfg = TcCfg<TN>;
  constexpr uint32_t kBStage = Cfg::kBStage, kColSfa = Cfg::kColSfa, kColSfb = Cfg::kColSfb, kColMeta = Cfg::kColMeta;
  constexpr int kStages = Cfg::kStages;
  constexpr int kTN = TN;
  extern __shared__ uint8_t tc_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(tc_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* a_s = base;                      // kStages x 4 KB
  uint8_t* b_s = base + kStages * kAStage;  // kStages x 16 KB
  __shared__ __align__(8) unsigned long long full[kStages], empty[kStages], acc_full[2], acc_empty[2], a_ready;
  __shared__ uint32_t tmem_base;
  __shared__ uint32_t code_a[16], code_m[16];
  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31u;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tmem_base)),
                 "n"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid < 16) {
    const BinCode c = bin_code(tid);
    code_a[tid] = c.abytes;
    code_m[tid] = c.meta;
  }
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(su32(&full[s]), 1);   // the loader's expect_tx arrival (+ the two copies' bytes)
      mbar_init(su32(&empty[s]), 1);  // the MMA commit
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(su32(&acc_full[a]), 1);
      mbar_init(su32(&acc_empty[a]), 4);
    }
    mbar_init(su32(&a_ready), 4);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  if (warp < 4) {  // scale factors: every byte 0x38 (ue4m3 1.0) over the SF columns of this warp's lanes
    const uint32_t lb = (warp * 32u) << 16;
    for (uint32_t c = kColSfa; c < kColMeta; c += 8) {
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %1, %1, %1, %1, %1, %1, %1};" ::"r"(tmem + lb + c),
                   "r"(0x38383838u));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");

  uint4* scr = p.scratch + static_cast<uint64_t>(blockIdx.x) * p.ksteps * (kAStage / 16);
  const uint64_t mtiles = (p.rows + kTM - 1) / kTM;
  const float half = 0.5f * static_cast<float>(p.F);
  uint32_t it = 0;     // global K-step counter (stage = it % kStages, phase = (it / kStages) & 1)
  uint32_t acc_n = 0;  // accumulators produced (acc_full / acc_empty phases)
  uint32_t tile_n = 0; // M tiles started (a_ready phase)
  for (uint64_t mt = blockIdx.x; mt < mtiles; mt += gridDim.x, ++tile_n) {
    const uint64_t r0 = mt * kTM;
    if (warp < 4) {
      // ---- A for every K step of this tile: L2 scratch (values) + TMEM (metadata) ----
      // (the previous tile's last accumulator was drained by these warps, so
      // every MMA reading the old scratch and metadata has completed)
      const uint32_t lb = (warp * 32u) << 16;
      const uint64_t r = r0 + tid;
      const bool rok = r < p.rows;
      const uint8_t* rowb = p.bins8 + (rok ? r : 0) * p.ldb;
      for (uint32_t ks = 0; ks < p.ksteps; ++ks) {
        uint2 bb = make_uint2(0xFFFFFFFFu, 0xFFFFFFFFu);
        if (rok) bb = __ldg(reinterpret_cast<const uint2*>(rowb + ks * 8u));
        uint32_t aw[8], m0 = 0, m1 = 0;
#pragma unroll
        for (uint32_t j = 0; j < 8; ++j) {
          const uint32_t b = ((j < 4 ? bb.x : bb.y) >> (8 * (j & 3))) & 0xFFu;
          const bool on = b < 16u && ks * 8u + j < p.F;  // bytes past F (row padding) are not features
          aw[j] = on ? code_a[b] : 0u;
          const uint32_t m = on ? code_m[b] : 0x44u;  // empty feature: both groups keep pairs (0, 1)
          if (j < 4) m0 |= m << (8 * j); else m1 |= m << (8 * (j - 4));
        }
        uint4* ap = scr + ks * (kAStage / 16) + (tid / 8) * 16 + (tid % 8);
        ap[0] = make_uint4(aw[0], aw[1], aw[2], aw[3]);
        ap[8] = make_uint4(aw[4], aw[5], aw[6], aw[7]);
        asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};" ::"r"(tmem + lb + kColMeta + 2 * ks),
                     "r"(m0), "r"(m1));
      }
      asm volatile("tcgen05.wait::st.sync.aligned;");
      asm volatile("fence.proxy.async.global;");  // the bulk copies (async proxy) read the scratch
      __threadfence();
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (lane == 0) mbar_arrive(su32(&a_ready));
    }
    for (uint32_t nt = 0; nt < p.ntiles; ++nt) {
      if (warp < 4) {
        // ---- epilogue: counts -> majority bits ----
        const uint32_t lb = (warp * 32u) << 16;
        const uint32_t ab = acc_n & 1u;  // this N tile's accumulator
        mbar_wait(su32(&acc_full[ab]), (acc_n >> 1) & 1u);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint64_t r = r0 + tid;
        for (uint32_t c0 = 0; c0 < ((p.ablate & 4u) ? 0u : static_cast<uint32_t>(kTN)); c0 += 32) {
          uint32_t v[32];
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
              "%14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
              : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
                "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]),
                "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]),
                "=r"(v[30]), "=r"(v[31])
              : "r"(tmem + lb + ab * kTN + c0));
          asm volatile("tcgen05.wait::ld.sync.aligned;");
          const uint32_t w = nt * (kTN / 32) + c0 / 32;
          if (w < p.W && r < p.rows) {
            const uint32_t t = __ldg(p.tie + w);
            uint32_t word = 0;
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              const float cnt = __uint_as_float(v[i]);
              const uint32_t bit = (cnt > half) || (cnt == half && ((t >> i) & 1u));
              word |= bit << i;
            }
            p.out[r * p.ldo + w] = word & valid_mask(w, p.D);
          }
        }
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncwarp();
        if (lane == 0) mbar_arrive(su32(&acc_empty[ab]));
      } else if (warp == 4) {
        // ---- loader: (A image, bound-table image) per K step ----
        if (lane == 0) {
          if (nt == 0) mbar_wait(su32(&a_ready), tile_n & 1u);
          for (uint32_t ks = 0; ks < p.ksteps; ++ks) {
            const uint32_t i = it + ks, s = i % kStages, ph = (i / kStages) & 1u;
            if (i >= kStages) mbar_wait(su32(&empty[s]), ph ^ 1u);
            const uint32_t fm = su32(&full[s]);
            if (p.ablate & 1u) {
              mbar_arrive(fm);
              continue;
            }
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(fm), "r"(kAStage + kBStage)
                         : "memory");
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    su32(a_s + s * kAStage)),
                "l"(scr + ks * (kAStage / 16)), "r"(kAStage), "r"(fm)
                : "memory");
            const uint4* src = p.img + (static_cast<uint64_t>(nt) * p.ksteps + ks) * (kBStage / 16);
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    su32(b_s + s * kBStage)),
                "l"(src), "r"(kBStage), "r"(fm)
                : "memory");
          }
        }
      } else {
        // ---- MMA issuer ----
        if (lane == 0) {
          const bool pf = p.prof != nullptr && blockIdx.x == 0;
          long long c0 = pf ? clock64() : 0;
          if (nt == 0) mbar_wait(su32(&a_ready), tile_n & 1u);                   // this tile's metadata is in TMEM
          if (pf) { const long long c1 = clock64(); p.prof[3] += c1 - c0; c0 = c1; }
          const uint32_t ab = acc_n & 1u;
          if (acc_n >= 2) mbar_wait(su32(&acc_empty[ab]), ((acc_n >> 1) - 1) & 1u);  // its previous use was drained
          if (pf) { const long long c1 = clock64(); p.prof[2] += c1 - c0; c0 = c1; }
          asm volatile("tcgen05.fence::after_thread_sync;");
          const uint32_t idesc = (1u << 2) | (1u << 7) | (1u << 10) | ((kTN >> 3) << 17) | ((kTM >> 4) << 24);
          // stage descriptors: the start-address field (bits 0-13, 16-byte units) advances by the stage size
          const uint64_t da0 = make_desc(su32(a_s), 128, 256), db0 = make_desc(su32(b_s), 128, 512);
          const uint32_t dacc = tmem + ab * kTN, sfa = tmem + kColSfa, sfb = tmem + kColSfb;
          uint32_t meta = tmem + kColMeta;
          uint32_t s = it % kStages, ph = (it / kStages) & 1u;
          uint64_t da = da0 + s * (kAStage >> 4), db = db0 + s * (kBStage >> 4);
          uint32_t fb = su32(&full[s]), eb = su32(&empty[s]);
          // one asm block per K step: wait for the stage, issue, commit the stage back to the loader
          // (no tcgen05 fence per step: the stage's data arrives through the async proxy; the TMEM
          // metadata was ordered once, after the a_ready wait)
          for (uint32_t ks = 0; ks < p.ksteps; ++ks) {
            const uint32_t acc = ks > 0 ? 1u : 0u;
            asm volatile(
                "{\n\t.reg .pred p, q;\n\tWAIT_%=:\n\t"
                "mbarrier.try_wait.parity.shared::cta.b64 p, [%8], %9;\n\t@!p bra WAIT_%=;\n\t"
                "setp.ne.b32 q, %4, 0;\n\t"
                "tcgen05.mma.sp.cta_group::1.kind::mxf4nvf4.block_scale.block16 [%0], %1, %2, [%7], %3, [%5], [%6], "
                "q;\n\t"
                "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%10];\n\t}\n" ::"r"(dacc),
                "l"(da), "l"(db), "r"(idesc), "r"(acc), "r"(sfa), "r"(sfb), "r"(meta), "r"(fb), "r"(ph), "r"(eb)
                : "memory");
            meta += 2u;
            if (++s == static_cast<uint32_t>(kStages)) {
              s = 0;
              ph ^= 1u;
              da = da0;
              db = db0;
              fb = su32(&full[0]);
              eb = su32(&empty[0]);
            } else {
              da += kAStage >> 4;
              db += kBStage >> 4;
              fb += 8u;
              eb += 8u;
            }
          }
          if (pf) { const long long c1 = clock64(); p.prof[4] += c1 - c0; c0 = c1; }
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                           su32(&acc_full[ab]))
                       : "memory");
        }
      }
      it += p.ksteps;
      ++acc_n;
      __syncwarp();
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kTmemCols));
}

}  // namespace

// The tensor-core encoder: ID-level binding, whole rows, B <= 16 bins. Returns
// false (nothing launched) when the shape is not supported.
namespace {
template <int TN>
void launch_tc_n(hv_context* ctx, cudaStream_t st, const uint8_t* bins8, uint32_t ldb, uint64_t rows, uint32_t F,
                 const uint32_t* id, const uint32_t* val, uint32_t B, uint32_t D, uint32_t W, const uint32_t* tie,
                 uint32_t* out, uint32_t ldo, uint32_t ksteps, size_t smem) {
  using Cfg = TcCfg<TN>;
  const uint32_t ntiles = (D + TN - 1) / TN;
  const uint64_t mtiles = (rows + kTM - 1) / kTM;
  const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(mtiles, static_cast<uint64_t>(ctx->sm_count)));
  DevBuf<uint4> img(static_cast<size_t>(ntiles) * ksteps * (Cfg::kBStage / 16), st);
  DevBuf<uint4> scratch(static_cast<size_t>(grid) * ksteps * (kAStage / 16), st);
  {
    const uint64_t total = static_cast<uint64_t>(ntiles) * ksteps * TN * 4;
    const unsigned tg = static_cast<unsigned>(std::min<uint64_t>((total + 255) / 256, 148ull * 16));
    tc_table_kernel<TN><<<tg, 256, 0, st>>>(id, val, F, B, D, W, ksteps, ntiles, img.ptr);
    launched("tc_table_kernel");
  }
  ck(cudaFuncSetAttribute(encode_tc_kernel<TN>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)),
     "cudaFuncSetAttribute");
  TcParams p{bins8, ldb, rows, F, D, W, ksteps, ntiles, img.ptr, scratch.ptr, tie, out, ldo ? ldo : W, 0u, nullptr};
  if (const char* ab = getenv("HVB200_TC_ABLATE")) p.ablate = static_cast<uint32_t>(atoi(ab));
  const char* pe = getenv("HVB200_TC_PROF");
  DevBuf<unsigned long long> prof(pe && pe[0] == '1' ? 8 : 0, st);
  if (prof.ptr) {
    prof.zero();
    p.prof = prof.ptr;
  }
  const long long t0 = 0;
  (void)t0;
  encode_tc_kernel<TN><<<grid, kThreads, smem, st>>>(p);
  launched("encode_tc_kernel");
  if (prof.ptr) {
    unsigned long long h[8];
    ck(cudaMemcpyAsync(h, prof.ptr, sizeof(h), cudaMemcpyDeviceToHost, st), "D2H");
    ck(cudaStreamSynchronize(st), "sync");
    const double mmas = static_cast<double>((rows + kTM - 1) / kTM / grid) * ntiles * ksteps;
    fprintf(stderr, "encode_tc CTA 0 MMA thread, cycles per UMMA: full-wait %.1f, acc-wait %.1f, a_ready-wait %.1f, issue %.1f\n",
            h[1] / mmas, h[2] / mmas, h[3] / mmas, h[4] / mmas);
  }
}
}  // namespace

bool launch_tc(hv_context* ctx, cudaStream_t st, const uint8_t* bins8, uint32_t ldb, uint64_t rows, uint32_t F,
               const uint32_t* id, const uint32_t* val, uint32_t B, uint32_t D, uint32_t W, const uint32_t* tie,
               uint32_t* out, uint32_t ldo) {
  if (B > 16u || F == 0 || rows == 0 || D == 0) return false;
  const uint32_t ksteps = (F + 7) / 8;
  if (ldb < ksteps * 8u || (ldb % 8) != 0 || (reinterpret_cast<uintptr_t>(bins8) & 7u)) return false;
  // N = 192 (two accumulators) while the tile's metadata fits beside them, else N = 128
  const char* nenv = getenv("HVB200_TC_N");  // evaluation: force N = 128
  const bool wide = ksteps <= TcCfg<192>::kMaxKsteps && !(nenv && atoi(nenv) == 128);
  if (!wide && ksteps > TcCfg<128>::kMaxKsteps) return false;
  const uint32_t bstage = wide ? TcCfg<192>::kBStage : TcCfg<128>::kBStage;
  const size_t smem = 1024 + static_cast<size_t>(wide ? TcCfg<192>::kStages : TcCfg<128>::kStages) * (kAStage + bstage);
  if (smem > ctx->smem_optin) return false;
  if (wide) {
    launch_tc_n<192>(ctx, st, bins8, ldb, rows, F, id, val, B, D, W, tie, out, ldo, ksteps, smem);
  } else {
    launch_tc_n<128>(ctx, st, bins8, ldb, rows, F, id, val, B, D, W, tie, out, ldo, ksteps, smem);
  }
  return true;
}

}  // namespace hvb
