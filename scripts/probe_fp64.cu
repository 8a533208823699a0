// Microbenchmark (not product code): fp64 add latency on this GPU — one
// dependent __dadd_rn chain per thread, one warp per SM (latency), and the
// same with a select feeding each add (the online replay's step shape).
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o probe_fp64 scripts/probe_fp64.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__global__ void chain(int iters, const double* __restrict__ v, double* out, long long* cyc) {
  double a = threadIdx.x * 1e-3;
  const double x = v[threadIdx.x & 7], y = v[(threadIdx.x + 3) & 7];
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) a = __dadd_rn(a, (u & 1) ? x : y);
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = a;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

__global__ void chain_sel(int iters, const uint32_t* __restrict__ words, const double* __restrict__ v, double* out,
                          long long* cyc) {
  __shared__ uint32_t sw[1024];
  __shared__ double sv[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) {
    sw[i] = words[i];
    sv[i] = v[i & 7] * (i + 1);
  }
  __syncthreads();
  double a = 0.0;
  const uint32_t lane = threadIdx.x & 31;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll 8
    for (int k = 0; k < 1024; ++k) {
      const double val = sv[k];
      const uint32_t wd = sw[k];
      a = __dadd_rn(a, ((wd >> lane) & 1u) ? val : 0.0);
    }
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = a;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

// the same step with the add predicated on the bit instead of selecting +0.0
__global__ void chain_pred(int iters, const uint32_t* __restrict__ words, const double* __restrict__ v, double* out,
                           long long* cyc) {
  __shared__ uint32_t sw[1024];
  __shared__ double sv[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) {
    sw[i] = words[i];
    sv[i] = v[i & 7] * (i + 1);
  }
  __syncthreads();
  double a = 0.0;
  const uint32_t lane = threadIdx.x & 31;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll 8
    for (int k = 0; k < 1024; ++k) {
      const double val = sv[k];
      const uint32_t wd = sw[k];
      if ((wd >> lane) & 1u) a = __dadd_rn(a, val);
    }
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = a;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

int main() {
  double *v, *out;
  uint32_t* w;
  long long* cyc;
  cudaMalloc(&v, 1024 * 8);
  cudaMalloc(&w, 1024 * 4);
  cudaMalloc(&out, 1 << 20);
  cudaMalloc(&cyc, 8);
  double hv[1024];
  uint32_t hw[1024];
  for (int i = 0; i < 1024; ++i) {
    hv[i] = 0.001 * (i + 1);
    hw[i] = 0x9E3779B9u * (i + 1);
  }
  cudaMemcpy(v, hv, sizeof hv, cudaMemcpyHostToDevice);
  cudaMemcpy(w, hw, sizeof hw, cudaMemcpyHostToDevice);
  long long c;
  for (int warps : {1, 2, 4, 8}) {
    chain<<<1, 32 * warps>>>(1000, v, out, cyc);
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("dependent DADD chain, %d warp(s)/SM: %.2f cycles per add\n", warps, c / (1000.0 * 16));
  }
  for (int warps : {1, 2, 8}) {
    chain_sel<<<1, 32 * warps>>>(20, w, v, out, cyc);
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("replay step (LDS word + LDS value + select + DADD), %d warp(s): %.2f cycles per step\n", warps,
           c / (20.0 * 1024));
  }
  for (int warps : {1, 2, 8}) {
    chain_pred<<<1, 32 * warps>>>(20, w, v, out, cyc);
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("replay step, predicated DADD, %d warp(s): %.2f cycles per step\n", warps, c / (20.0 * 1024));
  }
  return 0;
}
