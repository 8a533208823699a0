// Microbenchmark (not product code): variants of the two HBM-streaming kernels
// — classical column counts and the few-class Hamming scan — at the CHB-MIT
// shape (W = 313 words per row, rows only 4-byte aligned), to pick load width,
// loads in flight, cache hints and grid shape with CUDA-event timing.
//
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o probe_stream scripts/probe_stream.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <vector>

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e = (x);                                                             \
    if (e != cudaSuccess) {                                                          \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      return 1;                                                                      \
    }                                                                                \
  } while (0)

__device__ __forceinline__ void csa(uint32_t& h, uint32_t& l, uint32_t a, uint32_t b, uint32_t c) {
  const uint32_t u = a ^ b;
  h = (a & b) | (u & c);
  l = u ^ c;
}

struct HS {
  uint32_t ones = 0, twos = 0, fours = 0, eights = 0, hi[8] = {};
  __device__ __forceinline__ void add16(const uint32_t* x) {
    uint32_t tA, tB, fA, fB, eA, eB, s16;
    csa(tA, ones, ones, x[0], x[1]);
    csa(tB, ones, ones, x[2], x[3]);
    csa(fA, twos, twos, tA, tB);
    csa(tA, ones, ones, x[4], x[5]);
    csa(tB, ones, ones, x[6], x[7]);
    csa(fB, twos, twos, tA, tB);
    csa(eA, fours, fours, fA, fB);
    csa(tA, ones, ones, x[8], x[9]);
    csa(tB, ones, ones, x[10], x[11]);
    csa(fA, twos, twos, tA, tB);
    csa(tA, ones, ones, x[12], x[13]);
    csa(tB, ones, ones, x[14], x[15]);
    csa(fB, twos, twos, tA, tB);
    csa(eB, fours, fours, fA, fB);
    csa(s16, eights, eights, eA, eB);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const uint32_t t = hi[k] & s16;
      hi[k] ^= s16;
      s16 = t;
    }
  }
  __device__ __forceinline__ uint32_t count_of(int t) const {
    uint32_t c = ((ones >> t) & 1u) | (((twos >> t) & 1u) << 1) | (((fours >> t) & 1u) << 2) | (((eights >> t) & 1u) << 3);
#pragma unroll
    for (int k = 0; k < 8; ++k) c |= ((hi[k] >> t) & 1u) << (4 + k);
    return c;
  }
};

template <int LT>
__device__ __forceinline__ uint32_t ld(const uint32_t* p) {
  if constexpr (LT == 0) return __ldcs(p);
  else if constexpr (LT == 1) return __ldg(p);
  else return *p;
}

// A: round-1 kernel (thread per column, 32 rows in flight, blockIdx.y = chunk)
__global__ void __launch_bounds__(128) cc_old(const uint32_t* __restrict__ m, uint32_t W, const uint32_t* __restrict__ perm,
                                              uint64_t npos, uint32_t chunk, uint32_t* counts) {
  const uint32_t w = blockIdx.x * blockDim.x + threadIdx.x;
  const bool active = w < W;
  uint64_t p0 = static_cast<uint64_t>(blockIdx.y) * chunk;
  if (p0 >= npos) return;
  const uint64_t e = min(npos, p0 + chunk);
  HS h;
  uint32_t rows_nx[32];
#pragma unroll
  for (int t = 0; t < 32; ++t) rows_nx[t] = p0 + t < e ? perm[p0 + t] : 0u;
  for (uint64_t p = p0; p < e; p += 32) {
    uint32_t rr[32];
#pragma unroll
    for (int t = 0; t < 32; ++t) rr[t] = rows_nx[t];
    uint32_t x[32];
#pragma unroll
    for (int t = 0; t < 32; ++t) x[t] = (active && p + t < e) ? m[static_cast<uint64_t>(rr[t]) * W + w] : 0u;
    if (p + 32 < e) {
#pragma unroll
      for (int t = 0; t < 32; ++t) rows_nx[t] = p + 32 + t < e ? perm[p + 32 + t] : 0u;
    }
    h.add16(x);
    h.add16(x + 16);
  }
  if (active)
    for (int t = 0; t < 32; ++t) {
      const uint32_t c = h.count_of(t);
      if (c) atomicAdd(counts + 32 * w + t, c);
    }
}

// B: warp item = (chunk, 32*K-word group); lane owns K columns, R rows per batch
template <int K, int R, int LT>
__global__ void __launch_bounds__(128) cc_new(const uint32_t* __restrict__ m, uint32_t W, const uint32_t* __restrict__ perm,
                                              uint64_t npos, uint32_t chunk, uint32_t* counts, uint32_t ldm = 0) {
  if (ldm == 0) ldm = W;
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t groups = (W + 32 * K - 1) / (32 * K);
  const uint64_t items = (npos + chunk - 1) / chunk * groups;
  const uint64_t nwarps = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t it = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; it < items; it += nwarps) {
    const uint32_t g = static_cast<uint32_t>(it % groups);
    const uint32_t col = g * (32 * K) + lane;
    const uint64_t p0 = (it / groups) * chunk;
    const uint64_t e = min(npos, p0 + chunk);
    bool ok[K];
#pragma unroll
    for (int k = 0; k < K; ++k) ok[k] = col + 32 * k < W;
    HS h[K];
    uint32_t nxt = 0;
    if (lane < R && p0 + lane < e) nxt = __ldg(perm + p0 + lane);
    for (uint64_t p = p0; p < e; p += R) {
      const uint32_t cur = nxt;
      const uint32_t nvalid = e - p < R ? static_cast<uint32_t>(e - p) : static_cast<uint32_t>(R);
      uint32_t x[K][R < 16 ? 16 : R];
#pragma unroll
      for (int t = 0; t < R; ++t) {
        const uint32_t r = __shfl_sync(0xFFFFFFFFu, cur, t);
        const uint32_t* base = m + static_cast<uint64_t>(r) * ldm + col;
#pragma unroll
        for (int k = 0; k < K; ++k) x[k][t] = (ok[k] && t < nvalid) ? ld<LT>(base + 32 * k) : 0u;
      }
      const uint64_t q = p + R + lane;
      if (lane < R && q < e) nxt = __ldg(perm + q);
      if constexpr (R >= 16) {
#pragma unroll
        for (int k = 0; k < K; ++k)
#pragma unroll
          for (int j = 0; j < R; j += 16) h[k].add16(&x[k][j]);
      } else {
#pragma unroll
        for (int k = 0; k < K; ++k) {
#pragma unroll
          for (int t = R; t < 16; ++t) x[k][t] = 0;
          h[k].add16(x[k]);
        }
      }
    }
#pragma unroll
    for (int k = 0; k < K; ++k) {
      if (!ok[k]) continue;
      for (int t = 0; t < 32; ++t) {
        const uint32_t c = h[k].count_of(t);
        if (c) atomicAdd(counts + 32 * (col + 32 * k) + t, c);
      }
    }
  }
}

// predict: warp per row, 2 classes, U words in flight per lane
template <int U, int LT>
__global__ void __launch_bounds__(256) pred2(const uint32_t* __restrict__ cv, uint32_t W, const uint32_t* __restrict__ enc,
                                             uint64_t rows, int32_t* labels) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint64_t stride = (uint64_t)gridDim.x * (blockDim.x >> 5);
  for (uint64_t r = blockIdx.x * (uint64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); r < rows; r += stride) {
    const uint32_t* q = enc + r * W;
    uint32_t a0 = 0, a1 = 0;
    for (uint32_t w0 = 0; w0 < W; w0 += 32u * U) {
      uint32_t x[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t w = w0 + lane + 32u * u;
        x[u] = w < W ? ld<LT>(q + w) : 0u;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t w = w0 + lane + 32u * u;
        if (w < W) {
          a0 += __popc(x[u] ^ __ldg(cv + w));
          a1 += __popc(x[u] ^ __ldg(cv + W + w));
        }
      }
    }
    a0 = __reduce_add_sync(0xFFFFFFFFu, a0);
    a1 = __reduce_add_sync(0xFFFFFFFFu, a1);
    if (lane == 0) labels[r] = a1 < a0 ? 1 : 0;
  }
}

// predict, two rows per warp (16 lanes per row), U words per lane
template <int U, int LT>
__global__ void __launch_bounds__(256) pred2h(const uint32_t* __restrict__ cv, uint32_t W, const uint32_t* __restrict__ enc,
                                              uint64_t rows, int32_t* labels) {
  const uint32_t lane = threadIdx.x & 15u, half = (threadIdx.x >> 4) & 1u;
  const uint64_t stride = (uint64_t)gridDim.x * (blockDim.x >> 5) * 2;
  for (uint64_t r0 = (blockIdx.x * (uint64_t)(blockDim.x >> 5) + (threadIdx.x >> 5)) * 2; r0 < rows; r0 += stride) {
    const uint64_t r = r0 + half;
    const bool live = r < rows;
    const uint32_t* q = enc + (live ? r : 0) * W;
    uint32_t a0 = 0, a1 = 0;
    for (uint32_t w0 = 0; w0 < W; w0 += 16u * U) {
      uint32_t x[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t w = w0 + lane + 16u * u;
        x[u] = (live && w < W) ? ld<LT>(q + w) : 0u;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t w = w0 + lane + 16u * u;
        if (w < W) {
          a0 += __popc(x[u] ^ __ldg(cv + w));
          a1 += __popc(x[u] ^ __ldg(cv + W + w));
        }
      }
    }
#pragma unroll
    for (int o = 8; o; o >>= 1) {
      a0 += __shfl_xor_sync(0xFFFFFFFFu, a0, o);
      a1 += __shfl_xor_sync(0xFFFFFFFFu, a1, o);
    }
    if (lane == 0 && live) labels[r] = a1 < a0 ? 1 : 0;
  }
}

// C: pitched rows (Wp = W rounded up to 4 words, 16-byte aligned): a lane owns
// 4 consecutive columns through one 16-byte load per row, R rows per batch
template <int R>
__global__ void __launch_bounds__(128) cc_pitched(const uint32_t* __restrict__ m, uint32_t W, uint32_t Wp,
                                                  const uint32_t* __restrict__ perm, uint64_t npos, uint32_t chunk,
                                                  uint32_t* counts) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t groups = (W + 127) / 128;
  const uint64_t items = (npos + chunk - 1) / chunk * groups;
  const uint64_t nwarps = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t it = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; it < items; it += nwarps) {
    const uint32_t g = static_cast<uint32_t>(it % groups);
    const uint32_t col = g * 128 + 4 * lane;
    const bool ok = col < W;
    const uint64_t p0 = (it / groups) * chunk;
    const uint64_t e = min(npos, p0 + chunk);
    HS h[4];
    uint32_t nxt = 0;
    if (lane < R && p0 + lane < e) nxt = __ldg(perm + p0 + lane);
    for (uint64_t p = p0; p < e; p += R) {
      const uint32_t cur = nxt;
      const uint32_t nvalid = e - p < R ? static_cast<uint32_t>(e - p) : static_cast<uint32_t>(R);
      uint32_t x[4][R < 16 ? 16 : R];
#pragma unroll
      for (int t = 0; t < R; ++t) {
        const uint32_t r = __shfl_sync(0xFFFFFFFFu, cur, t);
        uint4 v = make_uint4(0, 0, 0, 0);
        if (ok && t < nvalid) v = __ldg(reinterpret_cast<const uint4*>(m + static_cast<uint64_t>(r) * Wp + col));
        x[0][t] = v.x;
        x[1][t] = v.y;
        x[2][t] = v.z;
        x[3][t] = v.w;
      }
      const uint64_t q = p + R + lane;
      if (lane < R && q < e) nxt = __ldg(perm + q);
#pragma unroll
      for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int j = 0; j < R; j += 16) h[k].add16(&x[k][j]);
    }
    if (ok)
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (col + k >= W) continue;
        for (int t = 0; t < 32; ++t) {
          const uint32_t c = h[k].count_of(t);
          if (c) atomicAdd(counts + 32 * (col + k) + t, c);
        }
      }
  }
}

// predict on pitched rows: warp per row, a lane holds U uint4 (4U words)
template <int U>
__global__ void __launch_bounds__(256) pred2p(const uint32_t* __restrict__ cv, uint32_t W, uint32_t Wp,
                                              const uint32_t* __restrict__ enc, uint64_t rows, int32_t* labels) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint64_t stride = (uint64_t)gridDim.x * (blockDim.x >> 5);
  for (uint64_t r = blockIdx.x * (uint64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); r < rows; r += stride) {
    const uint4* q = reinterpret_cast<const uint4*>(enc + r * Wp);
    const uint32_t nv = Wp / 4;
    uint32_t a0 = 0, a1 = 0;
    for (uint32_t v0 = 0; v0 < nv; v0 += 32u * U) {
      uint4 x[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t v = v0 + lane + 32u * u;
        x[u] = v < nv ? __ldg(q + v) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t v = v0 + lane + 32u * u;
        if (v < nv) {
          const uint4 c0 = __ldg(reinterpret_cast<const uint4*>(cv) + v);
          const uint4 c1 = __ldg(reinterpret_cast<const uint4*>(cv + Wp) + v);
          a0 += __popc(x[u].x ^ c0.x) + __popc(x[u].y ^ c0.y) + __popc(x[u].z ^ c0.z) + __popc(x[u].w ^ c0.w);
          a1 += __popc(x[u].x ^ c1.x) + __popc(x[u].y ^ c1.y) + __popc(x[u].z ^ c1.z) + __popc(x[u].w ^ c1.w);
        }
      }
    }
    a0 = __reduce_add_sync(0xFFFFFFFFu, a0);
    a1 = __reduce_add_sync(0xFFFFFFFFu, a1);
    if (lane == 0) labels[r] = a1 < a0 ? 1 : 0;
  }
}

// read-bandwidth ceiling: every uint4 of a flat range, xor-reduced
__global__ void __launch_bounds__(256) read_all(const uint4* __restrict__ p, uint64_t n, uint32_t* out) {
  uint32_t acc = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint4 v = __ldg(p + i);
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x12345678u) out[0] = acc;
}

__global__ void fill_random(uint32_t* p, uint64_t n, uint64_t seed) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t x = (i + seed) * 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    p[i] = static_cast<uint32_t>(x ^ (x >> 31));
  }
}

template <class F>
float timeit(F f, int reps = 7) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();
  cudaDeviceSynchronize();
  std::vector<float> ts;
  for (int i = 0; i < reps; ++i) {
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    ts.push_back(ms);
  }
  std::sort(ts.begin(), ts.end());
  return ts[ts.size() / 2];
}

int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  const uint32_t W = 313;
  const uint64_t rows = 5648000;
  const uint64_t n = rows * W;
  uint32_t *m, *perm, *counts, *cv;
  int32_t* labels;
  CK(cudaMalloc(&m, rows * 320ull * 4));
  CK(cudaMalloc(&perm, rows * 4));
  CK(cudaMalloc(&counts, 32 * W * 4));
  CK(cudaMalloc(&cv, 2 * 316 * 4));
  CK(cudaMalloc(&labels, rows * 4));
  {
    std::vector<uint32_t> h(rows);
    // class-sorted permutation of CHB-MIT-like labels: 120-row positive runs every 40,000 rows
    uint64_t k = 0;
    for (uint64_t i = 0; i < rows; ++i)
      if (i % 40000 >= 120) h[k++] = static_cast<uint32_t>(i);
    for (uint64_t i = 0; i < rows; ++i)
      if (i % 40000 < 120) h[k++] = static_cast<uint32_t>(i);
    CK(cudaMemcpy(perm, h.data(), rows * 4, cudaMemcpyHostToDevice));
  }
  fill_random<<<1024, 256>>>(m, rows * 320ull, 1);
  CK(cudaDeviceSynchronize());
  CK(cudaMemset(cv, 0x33, 2 * W * 4));
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const double cc_bytes = rows * (4.0 * W + 4);
  const uint64_t prow = 1412000;
  const double p_bytes = prow * (4.0 * W + 4);
  auto report = [&](const char* name, float ms, double bytes) {
    const cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("%s: CUDA error %s\n", name, cudaGetErrorString(e));
      exit(1);
    }
    printf("%-40s %8.3f ms  %7.1f GB/s\n", name, ms, bytes / (ms / 1e3) / 1e9);
  };
  const uint32_t chunk = 2048;
  {
    dim3 g((W + 127) / 128, (rows + chunk - 1) / chunk);
    report("colcount old", timeit([&] { cc_old<<<g, 128>>>(m, W, perm, rows, chunk, counts); }), cc_bytes);
  }
#define CCV(K, R, LT, NAME)                                                                                 \
  {                                                                                                         \
    int per_sm = 0;                                                                                         \
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, cc_new<K, R, LT>, 128, 0);                       \
    const uint64_t items = (rows + chunk - 1) / chunk * ((W + 32 * K - 1) / (32 * K));                     \
    const uint64_t slots = (uint64_t)sms * per_sm * 4;                                                      \
    const uint64_t waves = (items + slots - 1) / slots;                                                     \
    const unsigned gw = (unsigned)(((items + waves - 1) / waves + 3) / 4);                                 \
    const unsigned g1 = (unsigned)((items + 3) / 4);                                                        \
    char nm[96];                                                                                            \
    snprintf(nm, sizeof nm, "%s waves (occ %d)", NAME, per_sm);                                             \
    report(nm, timeit([&] { cc_new<K, R, LT><<<gw, 128>>>(m, W, perm, rows, chunk, counts); }), cc_bytes);  \
    snprintf(nm, sizeof nm, "%s one-shot", NAME);                                                           \
    report(nm, timeit([&] { cc_new<K, R, LT><<<g1, 128>>>(m, W, perm, rows, chunk, counts); }), cc_bytes);  \
  }
  CCV(4, 16, 1, "cc K4 R16 ldg")
  CCV(2, 16, 1, "cc K2 R16 ldg")
  CCV(1, 32, 1, "cc K1 R32 ldg")
  CCV(1, 16, 1, "cc K1 R16 ldg")
#define PV(KER, U, LT, NAME)                                                                       \
  {                                                                                                \
    for (int bpsm : {4, 8, 16}) {                                                                  \
      char nm[96];                                                                                 \
      snprintf(nm, sizeof nm, "%s grid %d/SM", NAME, bpsm);                                        \
      report(nm, timeit([&] { KER<U, LT><<<sms * bpsm, 256>>>(cv, W, m, prow, labels); }), p_bytes); \
    }                                                                                              \
  }
  PV(pred2, 1, 2, "pred U1 plain")
  PV(pred2, 10, 1, "pred U10 ldg")
  PV(pred2, 4, 1, "pred U4 ldg")
  PV(pred2h, 20, 1, "pred half-warp U20 ldg")
  PV(pred2h, 10, 1, "pred half-warp U10 ldg")
  for (uint32_t ldm : {313u, 320u, 316u}) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, cc_new<1, 32, 1>, 128, 0);
    const uint64_t items = (rows + chunk - 1) / chunk * ((W + 31) / 32);
    char nm[96];
    snprintf(nm, sizeof nm, "cc K1 R32 pitch %u one-shot", ldm);
    report(nm, timeit([&] { cc_new<1, 32, 1><<<(items + 3) / 4, 128>>>(m, W, perm, rows, chunk, counts, ldm); }),
           rows * (4.0 * W + 4));
  }
  {
    const uint32_t Wp = 316;
    for (int bpsm : {4, 8, 16, 32}) {
      char nm[96];
      snprintf(nm, sizeof nm, "read_all uint4 grid %d/SM", bpsm);
      report(nm, timeit([&] { read_all<<<sms * bpsm, 256>>>(reinterpret_cast<const uint4*>(m), rows * Wp / 4, counts); }),
             rows * Wp * 4.0);
    }
#define CCP(R)                                                                                          \
  {                                                                                                     \
    int per_sm = 0;                                                                                     \
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, cc_pitched<R>, 128, 0);                      \
    const uint64_t items = (rows + chunk - 1) / chunk * ((W + 127) / 128);                             \
    char nm[96];                                                                                        \
    snprintf(nm, sizeof nm, "cc pitched uint4 R%d one-shot (occ %d)", R, per_sm);                       \
    report(nm, timeit([&] { cc_pitched<R><<<(items + 3) / 4, 128>>>(m, W, Wp, perm, rows, chunk, counts); }), \
           rows * (4.0 * Wp + 4));                                                                      \
  }
    CCP(16)
    CCP(32)
    CCP(8)
    for (int bpsm : {8, 16, 32}) {
      char nm[96];
      snprintf(nm, sizeof nm, "pred pitched U3 grid %d/SM", bpsm);
      report(nm, timeit([&] { pred2p<3><<<sms * bpsm, 256>>>(cv, W, Wp, m, prow, labels); }), prow * (4.0 * Wp + 4));
      snprintf(nm, sizeof nm, "pred pitched U2 grid %d/SM", bpsm);
      report(nm, timeit([&] { pred2p<2><<<sms * bpsm, 256>>>(cv, W, Wp, m, prow, labels); }), prow * (4.0 * Wp + 4));
    }
  }
  CK(cudaDeviceSynchronize());
  return 0;
}
