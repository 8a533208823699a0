// Microbenchmark (not product code): the online trainer's replay step
// (csrc/hv_online.cu replay_chunk, COLS = 1) in isolation — one dependent
// fp64 chain per thread over 1,024 staged rows, word-major words and values in
// shared memory exactly as the product stages them — in several step forms,
// at 4 and 8 warps per SM (1 and 2 per scheduler). Reports cycles per row
// (clock64, max over CTAs); the floor is the 8.07-cycle DADD latency
// (profiles/probe_fp64_r2.txt).
//
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o probe_replay scripts/probe_replay.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

constexpr int kRows = 1024;
constexpr int kPitch = kRows + 4;

enum Form { kSelect, kFma, kAndMask, kUncond, kSelect2, kTwoCols, kGroups, kMaskWalk, kMaskWalk4, kMaskWalkLow, kMaskWalkDB };

template <int FORM>
__global__ void replay(int iters, const uint32_t* __restrict__ gw, const double* __restrict__ gv, double* out,
                       long long* cyc) {
  extern __shared__ __align__(16) uint8_t sm[];
  uint32_t* words = reinterpret_cast<uint32_t*>(sm);
  double* val = reinterpret_cast<double*>(sm + 8 * kPitch * 4);
  const int nw = blockDim.x / 32;
  for (int i = threadIdx.x; i < nw * kPitch; i += blockDim.x) words[i] = gw[i % (8 * kPitch)];
  for (int i = threadIdx.x; i < kRows; i += blockDim.x) val[i] = gv[i];
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31u, ww = threadIdx.x >> 5;
  const uint32_t* wv = words + ww * kPitch;
  double acc = 0.0;
  // kMaskWalk: each lane's 32-row masks (bit 31 - r = row r of the window has
  // this lane's bit set), built by a shuffle transpose of the window's words;
  // stored in place of the words (the walk reads only the masks)
  uint32_t* tmask = words + 8 * kPitch + 2 * kRows + 64;  // past the values (+ one 0.0 sentinel)
  if constexpr (FORM == kMaskWalk || FORM == kMaskWalk4 || FORM == kMaskWalkLow || FORM == kMaskWalkDB) {
    for (uint32_t g = 0; g < kRows / 32; ++g) {
      // kMaskWalk(4): row 31 - lane, rows reversed so clz gives the next row; kMaskWalkLow: natural order
      uint32_t x = wv[g * 32 + (FORM == kMaskWalkLow || FORM == kMaskWalkDB ? lane : 31 - lane)];
#pragma unroll
      for (uint32_t st = 16; st >= 1; st >>= 1) {
        const uint32_t m = st == 16 ? 0x0000FFFFu : st == 8 ? 0x00FF00FFu : st == 4 ? 0x0F0F0F0Fu
                         : st == 2 ? 0x33333333u : 0x55555555u;
        const bool lo = (lane & st) == 0;
        const uint32_t y = __shfl_xor_sync(0xFFFFFFFFu, x, st);
        const uint32_t t = __funnelshift_l(y, y, lo ? st : 32 - st);
        const uint32_t km = lo ? m : ~m;
        x = (x & km) | (t & ~km);
      }
      tmask[(ww * (kRows / 32) + g) * 32 + lane] = x;
    }
    if (threadIdx.x == 0) val[kRows] = 0.0;
    __syncthreads();
  }
  // kMaskWalkDB: values permuted so the de Bruijn hash of a row's lowest-bit
  // word indexes it directly: vdb[g * 32 + ((1 << r) * 0x077CB531 >> 27)] = val[g * 32 + r]
  double* vdb = reinterpret_cast<double*>(tmask + 8 * kRows + 64);
  if constexpr (FORM == kMaskWalkDB) {
    for (int i = threadIdx.x; i < kRows; i += blockDim.x) vdb[(i & ~31) + (((1u << (i & 31)) * 0x077CB531u) >> 27)] = val[i];
    if (threadIdx.x == 0) vdb[kRows] = 0.0;
    __syncthreads();
  }
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if constexpr (FORM == kMaskWalkDB) {
      // full-rate ALU only: lb = lowest set bit, its de Bruijn hash indexes the
      // permuted values; an empty mask reads the 0.0 sentinel
      const uint32_t* tm = tmask + ww * (kRows / 32) * 32 + lane;
      for (uint32_t g = 0; g < kRows / 32; ++g) {
        uint32_t m = tm[g * 32];
        const uint32_t nb = (__reduce_max_sync(0xFFFFFFFFu, __popc(m)) + 3u) / 4u;
        const double* vg = vdb + g * 32;
        auto pop = [&]() -> double {
          const uint32_t t = m - 1u;
          const uint32_t lb = m & ~t;
          m &= t;
          const double* a = lb ? vg + ((lb * 0x077CB531u) >> 27) : vdb + kRows;
          return *a;
        };
        double n0 = pop(), n1 = pop(), n2 = pop(), n3 = pop();
#pragma unroll 1
        for (uint32_t b = 0; b < nb; ++b) {
          const double v0 = n0, v1 = n1, v2 = n2, v3 = n3;
          n0 = pop();
          n1 = pop();
          n2 = pop();
          n3 = pop();
          acc = __dadd_rn(acc, v0);
          acc = __dadd_rn(acc, v1);
          acc = __dadd_rn(acc, v2);
          acc = __dadd_rn(acc, v3);
        }
      }
    } else if constexpr (FORM == kMaskWalkLow) {
      // natural order: the loop-carried chain is m &= m - 1 (two ALU ops); the
      // index (ffs) hangs off it
      const uint32_t* tm = tmask + ww * (kRows / 32) * 32 + lane;
      for (uint32_t g = 0; g < kRows / 32; ++g) {
        uint32_t m = tm[g * 32];
        const uint32_t nb = (__reduce_max_sync(0xFFFFFFFFu, __popc(m)) + 3u) / 4u;
        const uint32_t base = g * 32;
        auto pop = [&]() -> double {
          const uint32_t idx = m ? base + __ffs(m) - 1u : kRows;
          m &= m - 1u;
          return val[idx];
        };
        // two blocks of 4 in flight: the values added in block b were loaded
        // during block b - 2 (extra pops past the list read the 0.0 sentinel)
        double n0 = pop(), n1 = pop(), n2 = pop(), n3 = pop();
        double q0 = pop(), q1 = pop(), q2 = pop(), q3 = pop();
#pragma unroll 1
        for (uint32_t b = 0; b < nb; ++b) {
          const double v0 = n0, v1 = n1, v2 = n2, v3 = n3;
          n0 = q0;
          n1 = q1;
          n2 = q2;
          n3 = q3;
          q0 = pop();
          q1 = pop();
          q2 = pop();
          q3 = pop();
          acc = __dadd_rn(acc, v0);
          acc = __dadd_rn(acc, v1);
          acc = __dadd_rn(acc, v2);
          acc = __dadd_rn(acc, v3);
        }
      }
    } else if constexpr (FORM == kMaskWalk4) {
      // the walk in blocks of 4 pops (past the list: the 0.0 sentinel), the
      // next block's values loaded before this block's adds
      const uint32_t* tm = tmask + ww * (kRows / 32) * 32 + lane;
      for (uint32_t g = 0; g < kRows / 32; ++g) {
        uint32_t m = tm[g * 32];
        const uint32_t nb = (__reduce_max_sync(0xFFFFFFFFu, __popc(m)) + 3u) / 4u;
        const uint32_t base = g * 32;
        auto pop = [&]() -> double {
          const uint32_t r = __clz(m);
          const uint32_t idx = m ? base + r : kRows;
          m &= __funnelshift_rc(0x7FFFFFFFu, 0u, r);
          return val[idx];
        };
        double n0 = pop(), n1 = pop(), n2 = pop(), n3 = pop();
#pragma unroll 1
        for (uint32_t b = 0; b < nb; ++b) {
          const double v0 = n0, v1 = n1, v2 = n2, v3 = n3;
          if (b + 1 < nb) {
            n0 = pop();
            n1 = pop();
            n2 = pop();
            n3 = pop();
          }
          acc = __dadd_rn(acc, v0);
          acc = __dadd_rn(acc, v1);
          acc = __dadd_rn(acc, v2);
          acc = __dadd_rn(acc, v3);
        }
      }
    } else if constexpr (FORM == kMaskWalk) {
      // only the rows whose bit is set: per 32-row window, the warp's longest list
      const uint32_t* tm = tmask + ww * (kRows / 32) * 32 + lane;
      for (uint32_t g = 0; g < kRows / 32; ++g) {
        uint32_t m = tm[g * 32];
        const uint32_t cnt = __reduce_max_sync(0xFFFFFFFFu, __popc(m));
        const uint32_t base = g * 32;
#pragma unroll 4
        for (uint32_t i = 0; i < cnt; ++i) {
          const uint32_t r = __clz(m);
          const uint32_t idx = m ? base + r : kRows;
          m &= __funnelshift_rc(0x7FFFFFFFu, 0u, r);
          acc = __dadd_rn(acc, val[idx]);
        }
      }
    } else if constexpr (FORM == kGroups) {
      // the product's loop shape: 32-row groups, each skipped when its listed
      // mask (shared memory) is zero; every group listed here
      const uint32_t* gmask = words + 7 * kPitch;  // nonzero words
      for (uint32_t g = 0; g < kRows / 32; ++g) {
        if (gmask[g] == 0u) continue;
#pragma unroll
        for (uint32_t k = g * 32u; k < g * 32u + 32u; k += 4) {
          const uint4 w4 = *reinterpret_cast<const uint4*>(wv + k);
          const double2 v01 = *reinterpret_cast<const double2*>(val + k);
          const double2 v23 = *reinterpret_cast<const double2*>(val + k + 2);
          acc = __dadd_rn(acc, ((w4.x >> lane) & 1u) ? v01.x : 0.0);
          acc = __dadd_rn(acc, ((w4.y >> lane) & 1u) ? v01.y : 0.0);
          acc = __dadd_rn(acc, ((w4.z >> lane) & 1u) ? v23.x : 0.0);
          acc = __dadd_rn(acc, ((w4.w >> lane) & 1u) ? v23.y : 0.0);
        }
      }
    } else if constexpr (FORM == kTwoCols) {
      // two chains per thread: words ww and ww ^ 4 (another warp's word), one
      // shared stream of values
      const uint32_t* wv2 = words + (ww ^ 4u) * kPitch;
      double acc2 = 0.0;
#pragma unroll 8
      for (int k = 0; k < kRows; k += 4) {
        const uint4 w4 = *reinterpret_cast<const uint4*>(wv + k);
        const uint4 x4 = *reinterpret_cast<const uint4*>(wv2 + k);
        const double2 v01 = *reinterpret_cast<const double2*>(val + k);
        const double2 v23 = *reinterpret_cast<const double2*>(val + k + 2);
        acc = __dadd_rn(acc, ((w4.x >> lane) & 1u) ? v01.x : 0.0);
        acc2 = __dadd_rn(acc2, ((x4.x >> lane) & 1u) ? v01.x : 0.0);
        acc = __dadd_rn(acc, ((w4.y >> lane) & 1u) ? v01.y : 0.0);
        acc2 = __dadd_rn(acc2, ((x4.y >> lane) & 1u) ? v01.y : 0.0);
        acc = __dadd_rn(acc, ((w4.z >> lane) & 1u) ? v23.x : 0.0);
        acc2 = __dadd_rn(acc2, ((x4.z >> lane) & 1u) ? v23.x : 0.0);
        acc = __dadd_rn(acc, ((w4.w >> lane) & 1u) ? v23.y : 0.0);
        acc2 = __dadd_rn(acc2, ((x4.w >> lane) & 1u) ? v23.y : 0.0);
      }
      acc += acc2;
    } else if constexpr (FORM == kSelect2) {
      // addends of rows k+4..k+7 formed before the adds of rows k..k+3
      uint4 w4 = *reinterpret_cast<const uint4*>(wv);
      double2 a01 = *reinterpret_cast<const double2*>(val), a23 = *reinterpret_cast<const double2*>(val + 2);
      double s0 = ((w4.x >> lane) & 1u) ? a01.x : 0.0, s1 = ((w4.y >> lane) & 1u) ? a01.y : 0.0;
      double s2 = ((w4.z >> lane) & 1u) ? a23.x : 0.0, s3 = ((w4.w >> lane) & 1u) ? a23.y : 0.0;
#pragma unroll 8
      for (int k = 4; k < kRows + 4; k += 4) {
        const int kk = k < kRows ? k : 0;
        w4 = *reinterpret_cast<const uint4*>(wv + kk);
        a01 = *reinterpret_cast<const double2*>(val + kk);
        a23 = *reinterpret_cast<const double2*>(val + kk + 2);
        const double n0 = ((w4.x >> lane) & 1u) ? a01.x : 0.0, n1 = ((w4.y >> lane) & 1u) ? a01.y : 0.0;
        const double n2 = ((w4.z >> lane) & 1u) ? a23.x : 0.0, n3 = ((w4.w >> lane) & 1u) ? a23.y : 0.0;
        acc = __dadd_rn(acc, s0);
        acc = __dadd_rn(acc, s1);
        acc = __dadd_rn(acc, s2);
        acc = __dadd_rn(acc, s3);
        s0 = n0;
        s1 = n1;
        s2 = n2;
        s3 = n3;
      }
    } else {
#pragma unroll 8
      for (int k = 0; k < kRows; k += 4) {
        const uint4 w4 = *reinterpret_cast<const uint4*>(wv + k);
        const double2 v01 = *reinterpret_cast<const double2*>(val + k);
        const double2 v23 = *reinterpret_cast<const double2*>(val + k + 2);
        const uint32_t b[4] = {(w4.x >> lane) & 1u, (w4.y >> lane) & 1u, (w4.z >> lane) & 1u, (w4.w >> lane) & 1u};
        const double v[4] = {v01.x, v01.y, v23.x, v23.y};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if constexpr (FORM == kSelect) {
            acc = __dadd_rn(acc, b[u] ? v[u] : 0.0);
          } else if constexpr (FORM == kFma) {
            acc = __fma_rn(v[u], __hiloint2double(static_cast<int>(b[u] * 0x3FF00000u), 0), acc);
          } else if constexpr (FORM == kAndMask) {
            const int m = -static_cast<int>(b[u]);
            acc = __dadd_rn(acc, __hiloint2double(__double2hiint(v[u]) & m, __double2loint(v[u]) & m));
          } else {
            acc = __dadd_rn(acc, v[u]);
            (void)b;
          }
        }
      }
    }
  }
  const long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) atomicMax(reinterpret_cast<unsigned long long*>(cyc), static_cast<unsigned long long>(t1 - t0));
}

template <int FORM>
void run(const char* name, int sms, const uint32_t* w, const double* v, double* out, long long* cyc) {
  const int iters = 20;
  const size_t smem = 8 * kPitch * 4 + kRows * 8 + 64 * 4 + 8 * kRows * 4 + 64 * 4 + kRows * 8 + 64;
  cudaFuncSetAttribute(replay<FORM>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  for (int warps : {2, 3, 4, 5, 6, 8}) {
    cudaMemset(cyc, 0, 8);
    replay<FORM><<<sms, 32 * warps, smem>>>(iters, w, v, out, cyc);
    long long c = 0;
    cudaError_t e = cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) {
      printf("%s: %s\n", name, cudaGetErrorString(e));
      return;
    }
    static double h[256];
    cudaMemcpy(h, out, sizeof h, cudaMemcpyDeviceToHost);
    unsigned long long hs = 0;
    for (int i = 0; i < 32 * warps && i < 256; ++i) hs = hs * 1000003ull ^ reinterpret_cast<unsigned long long&>(h[i]);
    printf("%-34s %d warps/SM: %6.2f cycles per row (result hash %016llx)\n", name, warps, c / (double(iters) * kRows), hs);
  }
}

// The product's structure: a 288-thread CTA, warps 0-3 replay (one chain per
// thread) 256-row chunks with a CTA barrier after each, the other five warps
// only wait at the barriers; words word-major (pitch 260) and values in
// separate 256-row buffers.
__global__ void __launch_bounds__(288, 2) replay_cta(int iters, const uint32_t* __restrict__ gw,
                                                     const double* __restrict__ gv, double* out, long long* cyc,
                                                     double acc0, int nreplay, unsigned* done) {
  if (static_cast<int>(blockIdx.x) >= nreplay) {
    // the cooperative kernel's CTAs with no replay item wait in a grid barrier:
    // thread 0 polls a global word with acquire loads (as cg::grid_group::sync)
    if (threadIdx.x == 0) {
      unsigned v;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(done) : "memory");
      } while (v < static_cast<unsigned>(nreplay));
    }
    __syncthreads();
    return;
  }
  __shared__ __align__(16) uint32_t words[2][8 * 260];
  __shared__ __align__(16) double val[2][256];
  for (int i = threadIdx.x; i < 2 * 8 * 260; i += blockDim.x) (&words[0][0])[i] = gw[i % (8 * kPitch)];
  for (int i = threadIdx.x; i < 512; i += blockDim.x) (&val[0][0])[i] = gv[i % kRows];
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  double acc = acc0 * (1.0 + threadIdx.x * 1e-9);
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    for (uint32_t ch = 0; ch < 4; ++ch) {
      const uint32_t buf = ch & 1u;
      if (warp < 4) {
        const uint32_t* wv = words[buf] + warp * 260;
        const double* v = val[buf];
#pragma unroll 1
        for (uint32_t g = 0; g < 8; g += 2) {
#pragma unroll
          for (uint32_t k = g * 32u; k < g * 32u + 64u; k += 4) {
            const uint4 w4 = *reinterpret_cast<const uint4*>(wv + k);
            const double2 v01 = *reinterpret_cast<const double2*>(v + k);
            const double2 v23 = *reinterpret_cast<const double2*>(v + k + 2);
            acc = __dadd_rn(acc, ((w4.x >> lane) & 1u) ? v01.x : 0.0);
            acc = __dadd_rn(acc, ((w4.y >> lane) & 1u) ? v01.y : 0.0);
            acc = __dadd_rn(acc, ((w4.z >> lane) & 1u) ? v23.x : 0.0);
            acc = __dadd_rn(acc, ((w4.w >> lane) & 1u) ? v23.y : 0.0);
          }
        }
      }
      __syncthreads();
    }
  }
  const long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) {
    atomicMax(reinterpret_cast<unsigned long long*>(cyc), static_cast<unsigned long long>(t1 - t0));
    __threadfence();
    atomicAdd(done, 1u);
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint32_t* w;
  double *v, *out;
  long long* cyc;
  cudaMalloc(&w, 8 * kPitch * 4);
  cudaMalloc(&v, kRows * 8);
  cudaMalloc(&out, size_t(sms) * 1024 * 8);
  cudaMalloc(&cyc, 8);
  static uint32_t hw[8 * kPitch];
  static double hv[kRows];
  for (int i = 0; i < 8 * kPitch; ++i) hw[i] = 0x9E3779B9u * (i + 1);
  for (int i = 0; i < kRows; ++i) hv[i] = 0.001 * (i + 1) * ((i & 3) ? 1 : -1);
  cudaMemcpy(w, hw, sizeof hw, cudaMemcpyHostToDevice);
  cudaMemcpy(v, hv, sizeof hv, cudaMemcpyHostToDevice);
  unsigned* done;
  cudaMalloc(&done, 4);
  for (int spin : {0, 35, 69}) {
    cudaMemset(cyc, 0, 8);
    cudaMemset(done, 0, 4);
    replay_cta<<<79 + spin, 288>>>(20, w, v, out, cyc, 3e6, 79, done);
    long long c = 0;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("product structure (288-thread CTA, 4 replay warps, 256-row chunks + barriers), 79 replay CTAs + %d CTAs "
           "polling a global word: %6.2f cycles per row\n", spin, c / (20.0 * 1024));
  }
  run<kMaskWalkDB>("mask walk, de Bruijn index (ALU only)", sms, w, v, out, cyc);
  run<kMaskWalkLow>("mask walk, m &= m - 1, pipelined", sms, w, v, out, cyc);
  run<kMaskWalk4>("mask walk, 4-pop blocks pipelined", sms, w, v, out, cyc);
  run<kMaskWalk>("mask walk (set bits only, per lane)", sms, w, v, out, cyc);
  run<kSelect>("select (product form)", sms, w, v, out, cyc);
  run<kGroups>("select, 32-row groups with skip test", sms, w, v, out, cyc);
  run<kSelect2>("select, addends one group ahead", sms, w, v, out, cyc);
  run<kTwoCols>("two chains per thread (per chain)", sms, w, v, out, cyc);
  run<kFma>("fma with 0/1 factor", sms, w, v, out, cyc);
  run<kAndMask>("addend = v AND mask", sms, w, v, out, cyc);
  run<kUncond>("unconditional add (floor, wrong)", sms, w, v, out, cyc);
  return 0;
}
