// Microbenchmark: legacy mma.sync m16n8k32 s8 throughput vs XOR+POPC on this GPU.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o probe scripts/probe_imma_popc.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void imma_loop(int iters, int* out) {
  uint32_t a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
  int c[8][4] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k)
      asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+r"(c[k][0]), "+r"(c[k][1]), "+r"(c[k][2]), "+r"(c[k][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  int s = 0;
  for (int k = 0; k < 8; ++k) s += c[k][0] + c[k][1] + c[k][2] + c[k][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void popc_loop(int iters, int* out) {
  uint32_t x[8];
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * (k + 3);
  uint32_t acc[8] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) { acc[k] += __popc(x[k] ^ i); }
  }
  int s = 0;
  for (int k = 0; k < 8; ++k) s += acc[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  int* out; cudaMalloc(&out, 148 * 8 * 1024 * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 20000;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    imma_loop<<<148 * 4, 256>>>(iters, out);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double ops = 2.0 * 16 * 8 * 32 * 8.0 * iters * (148 * 4 * 256 / 32);
    printf("IMMA m16n8k32 s8: %.1f TOPS (%.2f ms)\n", ops / ms / 1e9, ms);
    cudaEventRecord(e0);
    popc_loop<<<148 * 4, 256>>>(iters * 4, out);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double pc = 8.0 * iters * 4 * 148 * 4 * 256;
    printf("POPC: %.2f T popc/s = %.1f T bit-ops/s (%.2f ms)\n", pc / ms / 1e9, pc * 32 / ms / 1e9, ms);
  }
  return 0;
}
