// Microbenchmark (not product code): integer-pipe and shared-memory issue
// rates on this GPU, per SM and clock, for the encoder's ceiling model
// (LOP3 on the ALU pipe and LDS.64 table reads).
//
// Each kernel runs 8 independent dependency chains per thread, 1024 threads
// per CTA, enough CTAs to fill every SM several times; cycles are taken from
// clock64() per CTA (max over the CTAs resident on an SM is the SM's busy
// time), so the result is in ops / clk / SM independent of the clock. The
// SASS of each loop body is checked with cuobjdump (counts printed by
// scripts/ run wrapper), so the op count per iteration is known.
//
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o probe_alu scripts/probe_alu.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <vector>

enum Op { kLop3, kIadd3, kPrmt, kPopc, kImad, kShf, kLds64, kLds32 };

template <int OP>
__global__ void __launch_bounds__(1024) ops_kernel(int iters, uint32_t seed, uint32_t* out,
                                                   unsigned long long* t_start, unsigned long long* t_end,
                                                   unsigned* n_cta) {
  __shared__ uint2 tab[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) tab[i] = make_uint2(i * 0x9E3779B9u, i ^ seed);
  __syncthreads();
  uint32_t a[8], b[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    a[j] = (threadIdx.x + 1) * (j + 3) ^ seed;
    b[j] = (threadIdx.x * 7 + j) * 0x85EBCA6Bu;
  }
  const unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if constexpr (OP == kLop3) {
          asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a[j]) : "r"(b[j]), "r"(b[(j + u + 1) & 7]));
        } else if constexpr (OP == kIadd3) {
          asm volatile("add.u32 %0, %0, %1;" : "+r"(a[j]) : "r"(b[(j + u) & 7]));
        } else if constexpr (OP == kPrmt) {
          asm volatile("prmt.b32 %0, %0, %1, 0x7651;" : "+r"(a[j]) : "r"(b[(j + u) & 7]));
        } else if constexpr (OP == kPopc) {
          uint32_t t;
          asm volatile("popc.b32 %0, %1;" : "=r"(t) : "r"(a[j]));
          a[j] = t;  // chain through popc (values stay small but distinct per lane)
        } else if constexpr (OP == kImad) {
          asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[j]) : "r"(b[j]), "r"(b[(j + u + 1) & 7]));
        } else if constexpr (OP == kShf) {
          asm volatile("shf.l.wrap.b32 %0, %0, %1, %2;" : "+r"(a[j]) : "r"(b[j]), "r"(b[(j + u + 1) & 7]));
        } else if constexpr (OP == kLds64) {
          // conflict-free: lane-consecutive 8-byte entries, independent of the chain
          const uint2 v = tab[((i * 4 + u) * 256 + j * 32 + (threadIdx.x & 31)) & 4095];
          a[j] ^= v.x;
          b[j] ^= v.y;
        } else {
          const uint32_t v = reinterpret_cast<const uint32_t*>(tab)[((i * 4 + u) * 256 + j * 32 + (threadIdx.x & 31)) & 8191];
          a[j] ^= v;
        }
      }
    }
  }
  const unsigned long long t1 = clock64();
  uint32_t s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s ^= a[j] ^ b[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    atomicMin(t_start + smid, t0);
    atomicMax(t_end + smid, t1);
    atomicAdd(n_cta + smid, 1u);
  }
}

template <int OP>
double run(const char* name, int sms, int iters) {
  const int blocks = sms * 4, threads = 1024;
  uint32_t* out;
  unsigned long long *ts, *te;
  unsigned* nc;
  cudaMalloc(&out, blocks * threads * 4);
  cudaMalloc(&ts, 1024 * 8);
  cudaMalloc(&te, 1024 * 8);
  cudaMalloc(&nc, 1024 * 4);
  auto reset = [&] {
    cudaMemset(ts, 0xFF, 1024 * 8);
    cudaMemset(te, 0, 1024 * 8);
    cudaMemset(nc, 0, 1024 * 4);
  };
  reset();
  ops_kernel<OP><<<blocks, threads>>>(iters / 10, 1, out, ts, te, nc);  // warm-up
  cudaDeviceSynchronize();
  reset();
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  ops_kernel<OP><<<blocks, threads>>>(iters, 1, out, ts, te, nc);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  std::vector<unsigned long long> hs(1024), he(1024);
  std::vector<unsigned> hn(1024);
  cudaMemcpy(hs.data(), ts, 1024 * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(he.data(), te, 1024 * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(hn.data(), nc, 1024 * 4, cudaMemcpyDeviceToHost);
  // per SM: (CTAs it ran x ops per CTA) / (last end - first start) in its own clock
  const double ops_per_cta = double(threads) * iters * 32;
  double best = 0, sum = 0, span_sum = 0;
  int used = 0;
  for (int i = 0; i < 1024; ++i)
    if (hn[i]) {
      const double span = double(he[i] - hs[i]);
      const double r = hn[i] * ops_per_cta / span;
      best = std::max(best, r);
      sum += r;
      span_sum += span;
      ++used;
    }
  const double mean = sum / std::max(used, 1);
  const double clk_mhz = (span_sum / std::max(used, 1)) / (ms * 1e3);
  printf("%-8s %7.2f ops/clk/SM mean over %d SMs (max %.2f); kernel %.3f ms; SM clock ~%.0f MHz\n", name, mean,
         used, best, ms, clk_mhz);
  cudaFree(out);
  cudaFree(ts);
  cudaFree(te);
  cudaFree(nc);
  return mean;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<kLop3>("LOP3", sms, 20000);
  run<kIadd3>("IADD", sms, 20000);
  run<kPrmt>("PRMT", sms, 20000);
  run<kPopc>("POPC", sms, 5000);
  run<kImad>("IMAD", sms, 20000);
  run<kShf>("SHF", sms, 20000);
  run<kLds64>("LDS.64", sms, 5000);
  run<kLds32>("LDS.32", sms, 5000);
  return 0;
}
