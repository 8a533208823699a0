// Microbenchmark (not product code): tcgen05 tensor-core throughput on this
// B200 for the operand kinds a tensor-core ID-level encoder would use — the
// one-hot x bound-table GEMM of DESIGN.md §8 (A = one-hot bins, 1 in 16 per
// feature, 2:4-sparse; B = the bound table, 0/1 entries; counts <= F exact in
// fp32). One elected thread per CTA issues back-to-back UMMAs (M = 128,
// N = 256) accumulating into TMEM from shared-memory operands, one CTA per SM
// on every SM; operand contents are a fixed random pattern (the rate is what
// is measured, not the result). Reports dense-equivalent TFLOP/s = 2·M·N·K per
// instruction (K = the logical K: sparse instructions cover twice the stored K).
//
//   kind::f8f6f4 (e4m3)           dense K = 32
//   kind::mxf4nvf4 block16 (e2m1) dense K = 64,  sparse (.sp) K = 128
//
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o probe_tc_fp4 scripts/probe_tc_fp4.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

constexpr int kM = 128;
constexpr uint32_t kTmemCols = 512;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

// K-major, no swizzle: core matrices of 8 rows x 16 bytes
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (static_cast<uint64_t>((saddr & 0x3FFFFu) >> 4)) | (static_cast<uint64_t>(lbo >> 4) << 16) |
         (static_cast<uint64_t>(sbo >> 4) << 32) | (1ull << 46);
}

enum Kind { kF8Dense, kF4Dense, kF4Sparse, kF4SparseCommitEach, kF4SparseRing, kF4SparseA256, kF4SparseMetaCycle,
            kF4SparseRing16, kF4SparseRing30, kF4SparseValid, kF4SparseStages, kF4SparseSpinners, kF4SparseD192 };

template <int KIND, int kN = 256>
__global__ void __launch_bounds__(128, 1) tc_rate(int iters, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) unsigned long long done;
  __shared__ __align__(8) unsigned long long ring[8];
  __shared__ __align__(8) unsigned long long ring2[32];
  const uint32_t tid = threadIdx.x, warp = tid >> 5;
  // operands: A 128 rows x 64 B, B 256 rows x 64 B (enough for every kind's K step), random bytes
  uint8_t* a = sm;
  uint8_t* b = sm + (KIND == kF4SparseStages ? 4096 : 128 * 64);  // stages: A 4 KB + B 12 KB per 16 KB
  const uint32_t nbytes = KIND == kF4SparseStages ? 8u * 16384u : (128u + 256u) * 64u;
  for (uint32_t i = tid; i < nbytes; i += blockDim.x) {
    uint32_t x = (i + 1) * 0x9E3779B9u;
    x ^= x >> 13;
    // e2m1 nibbles 0 or 1.0 (0x2), e4m3 bytes 0 or 0x08: a 0/1 pattern like the encoder's
    sm[i] = KIND == kF8Dense ? ((x & 1) ? 0x08 : 0) : static_cast<uint8_t>(((x & 1) ? 0x2 : 0) | ((x & 2) ? 0x20 : 0));
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "n"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&done)));
    for (int r = 0; r < 8; ++r) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&ring[r])));
    for (int r = 0; r < 32; ++r) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&ring2[r])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  if (KIND == kF4SparseValid || KIND == kF4Dense) {
    // valid operands: scale factors 1.0 (ue4m3 0x38) over columns 256..383, metadata (idx0, idx1) = (0, 1)
    const uint32_t lb = (warp * 32u) << 16;
    for (uint32_t c = 256; c < 384; c += 8)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %1, %1, %1, %1, %1, %1, %1};" ::"r"(tmem + lb + c),
                   "r"(0x38383838u));
    for (uint32_t c = 384; c < 512; c += 8)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %1, %1, %1, %1, %1, %1, %1};" ::"r"(tmem + lb + c),
                   "r"(0x44444444u));
    asm volatile("tcgen05.wait::st.sync.aligned;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
  }
  unsigned long long t0 = 0, t1 = 0;
  if (KIND == kF4SparseSpinners && warp >= 1) {
    // three warps polling the completion barrier with try_wait while thread 0 issues
    asm volatile(
        "{\n\t.reg .pred p;\n\tSPIN_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t"
        "@!p bra SPIN_%=;\n\t}\n" ::"r"(smem_u32(&done))
        : "memory");
  }
  if (tid == 0) {
    // 8-row core matrices 16 B wide: LBO = next core matrix along K (8 rows x 16 B = 128 B), SBO = next 8 rows
    // the encoder's compressed A: 32 bytes per row, 8-row core-matrix groups 256 bytes apart
    const uint64_t da = KIND == kF4SparseA256 ? make_desc(smem_u32(a), 128, 256) : make_desc(smem_u32(a), 128, 64 * 8);
    const uint64_t db = make_desc(smem_u32(b), 128, 64 * 8);
    const uint32_t d = KIND == kF4SparseD192 ? tmem + 192 : tmem;  // accumulator: columns [0, 256) (or from 192)
    const uint32_t sfa = tmem + 256;       // scale factors / sparse metadata (contents arbitrary)
    const uint32_t sfb = tmem + 320;
    const uint32_t meta = KIND == kF4SparseMetaCycle ? tmem + 416 - 86 + 0 : tmem + 384;
    uint32_t idesc;
    if constexpr (KIND == kF8Dense) {
      idesc = (1u << 4) | ((kN >> 3) << 17) | ((kM >> 4) << 24);  // D f32, A/B e4m3, K-major
    } else {
      // block-scaled: A/B e2m1 (MXF4 format 1), scale format ue4m3 (0) for block16, M, N; sparse flag bit 2
      idesc = (1u << 7) | (1u << 10) | ((kN >> 3) << 17) | ((kM >> 4) << 24) | (KIND != kF4Dense ? (1u << 2) : 0u);
    }
    t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint32_t acc = i > 0 ? 1u : 0u;
      if constexpr (KIND == kF8Dense) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
            "l"(da), "l"(db), "r"(idesc), "r"(acc));
      } else if constexpr (KIND == kF4Dense) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::mxf4nvf4.block_scale.block16 [%0], %1, %2, %3, [%5], [%6], p;\n\t}\n" ::"r"(d),
            "l"(da), "l"(db), "r"(idesc), "r"(acc), "r"(sfa), "r"(sfb));
      } else {
        // kF4SparseStages: operands from 8 different 16 KB stages in turn (A 4 KB + B 12 KB), as a pipeline reads them
        const uint64_t so = KIND == kF4SparseStages ? static_cast<uint64_t>((i & 7) * 16384 >> 4) : 0ull;
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.sp.cta_group::1.kind::mxf4nvf4.block_scale.block16 [%0], %1, %2, [%7], %3, [%5], [%6], p;\n\t}\n" ::"r"(d),
            "l"(da + so), "l"(db + so), "r"(idesc), "r"(acc), "r"(sfa), "r"(sfb),
            "r"(KIND == kF4SparseMetaCycle ? meta + 2u * static_cast<uint32_t>(i % 43) : meta));
        if constexpr (KIND == kF4SparseCommitEach) {
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&ring[i & 7]))
                       : "memory");
        }
        if constexpr (KIND == kF4SparseRing16 || KIND == kF4SparseRing30) {
          constexpr int R = KIND == kF4SparseRing16 ? 16 : 30;
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&ring2[i % R]))
                       : "memory");
          if (i >= R - 1) {
            const int j = i - (R - 1);
            asm volatile(
                "{\n\t.reg .pred p;\n\tWAITQ_%=:\n\t"
                "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
                "@!p bra WAITQ_%=;\n\t}\n" ::"r"(smem_u32(&ring2[j % R])), "r"((j / R) & 1)
                : "memory");
          }
        }
        if constexpr (KIND == kF4SparseRing) {
          // a ring of 8 stages: commit to stage i % 8, and before issuing i + 8 wait for its completion
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&ring[i & 7]))
                       : "memory");
          if (i >= 7) {
            const int j = i - 7;  // wait for MMA j (issued 7 ago) before the next issue reuses its stage
            asm volatile(
                "{\n\t.reg .pred p;\n\tWAITR_%=:\n\t"
                "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
                "@!p bra WAITR_%=;\n\t}\n" ::"r"(smem_u32(&ring[j & 7])), "r"((j >> 3) & 1)
                : "memory");
          }
        }
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&done))
                 : "memory");
    asm volatile(
        "{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t"
        "@!p bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(&done))
        : "memory");
    t1 = clock64();
    atomicMax(cyc, t1 - t0);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kTmemCols));
}

template <int KIND, int kN = 256>
void run(const char* name, int sms, int logical_k, int iters = 20000) {
  unsigned long long* cyc;
  cudaMalloc(&cyc, 8);
  const size_t smem = (KIND == kF4SparseStages ? 8 * 16384 : (128 + 256) * 64) + 1024;
  cudaFuncSetAttribute(tc_rate<KIND, kN>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  float best_ms = 1e30f;
  unsigned long long c = 0;
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemset(cyc, 0, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    tc_rate<KIND, kN><<<sms, 128, smem>>>(iters, cyc);
    cudaEventRecord(e1);
    cudaError_t err = cudaEventSynchronize(e1);
    if (err != cudaSuccess || cudaGetLastError() != cudaSuccess) {
      printf("%-40s: %s\n", name, cudaGetErrorString(err));
      return;
    }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best_ms) {
      best_ms = ms;
      cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    }
  }
  const double flop = 2.0 * kM * kN * logical_k * static_cast<double>(iters) * sms;
  printf("%-40s: %.1f cycles per UMMA (M=128 N=%d K=%d), %.0f TFLOP/s dense-equivalent over %d SMs (%.3f ms)\n", name,
         static_cast<double>(c) / iters, kN, logical_k, flop / (best_ms * 1e-3) / 1e12, sms, best_ms);
  cudaFree(cyc);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<kF8Dense>("kind::f8f6f4 e4m3 dense", sms, 32);
  run<kF4Dense>("kind::mxf4nvf4 e2m1 dense (block16)", sms, 64);
  run<kF4Sparse>("kind::mxf4nvf4 e2m1 2:4 sparse (block16)", sms, 128);
  run<kF4SparseA256, 192>("sparse N=192, A layout SBO 256 (encoder)", sms, 128);
  run<kF4SparseMetaCycle, 192>("sparse N=192, metadata column per K step", sms, 128);
  run<kF4SparseValid, 192>("sparse N=192, valid SF (1.0) + metadata", sms, 128);
  run<kF4SparseStages, 192>("sparse N=192, 8 rotating operand stages", sms, 128);
  run<kF4SparseSpinners, 192>("sparse N=192, 3 warps polling an mbarrier", sms, 128);
  run<kF4SparseD192, 192>("sparse N=192, accumulator at TMEM column 192", sms, 128);
  run<kF4SparseValid, 256>("sparse N=256, valid SF (1.0) + metadata", sms, 128);
  run<kF4SparseRing16, 192>("sparse N=192, 16-deep commit/wait ring", sms, 128);
  run<kF4SparseRing30, 192>("sparse N=192, 30-deep commit/wait ring", sms, 128);
  run<kF4SparseCommitEach, 192>("sparse N=192, commit after every UMMA", sms, 128);
  run<kF4SparseRing, 192>("sparse N=192, 8-deep commit/wait ring", sms, 128);
  run<kF4Sparse, 128>("kind::mxf4nvf4 2:4 sparse N=128", sms, 128);
  run<kF4Sparse, 176>("kind::mxf4nvf4 2:4 sparse N=176", sms, 128);
  run<kF4Sparse, 192>("kind::mxf4nvf4 2:4 sparse N=192", sms, 128);
  run<kF4Sparse, 64>("kind::mxf4nvf4 2:4 sparse N=64", sms, 128);
  // sustained: ~0.5 s per launch (power / clock behaviour of a long encode)
  run<kF4Sparse>("kind::mxf4nvf4 2:4 sparse, 0.5 s launches", sms, 128, 5600000);
  run<kF4Dense>("kind::mxf4nvf4 dense, 0.5 s launches", sms, 64, 7000000);
  return 0;
}
