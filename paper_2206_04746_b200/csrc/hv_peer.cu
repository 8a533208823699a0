// hv_peer.cu — classical training's all-reduce fused into the count kernel,
// over peer memory (model.cpp:219-244).
//
// Every rank owns a shared buffer (CUDA IPC: cudaIpcGetMemHandle / open on
// the peers) holding its class counts and class row counts, double-buffered by
// epoch parity, plus one arrival flag per rank. The column-count kernel of a
// rank flushes its exact per-bit counts with system-scope atomics straight
// into EVERY rank's buffer (NVLink P2P on a multi-GPU box, local memory for
// ranks sharing a GPU), then signals each peer's flag with a release store;
// a one-thread kernel on each rank waits (acquire) until all flags carry the
// epoch. The sums are order-free integers, so every rank ends with exactly the
// counts an all-reduce would give — without a separate collective pass.
//
// Buffer reuse: a rank zeroes its parity-p counts only after binarising them
// (hv_dev_peer_release), and peers write parity p again only two epochs
// later, after waiting for this rank's flag of the epoch in between.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>

#include "hv_internal.cuh"

namespace hvb {
namespace {

__global__ void add_rows_peers_kernel(const uint32_t* __restrict__ hist, uint32_t C, uint64_t* const* dsts,
                                      uint32_t ndst) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < C * ndst; i += gridDim.x * blockDim.x) {
    const uint32_t c = i % C, d = i / C;
    if (hist[c]) atomicAdd_system(reinterpret_cast<unsigned long long*>(dsts[d] + c), hist[c]);
  }
}

__global__ void signal_peers_kernel(uint32_t* const* flags, uint32_t world, uint32_t rank, uint32_t epoch) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  __threadfence_system();  // this rank's counts (earlier kernels on the stream) before the flags
  for (uint32_t q = 0; q < world; ++q) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(flags[q] + rank), "r"(epoch) : "memory");
  }
}

__global__ void wait_peers_kernel(const uint32_t* flags, uint32_t world, uint32_t epoch,
                                  unsigned long long* err) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (uint32_t q = 0; q < world; ++q) {
    for (;;) {
      uint32_t v;
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flags + q) : "memory");
      if (static_cast<int32_t>(v - epoch) >= 0) break;
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > 20000000000ull) {  // 20 s: a peer is gone; fail instead of hanging the GPU
        latch(err, kErrCount, q);
        return;
      }
      __nanosleep(256);
    }
  }
  __threadfence_system();
}

}  // namespace
}  // namespace hvb

using namespace hvb;

extern "C" {

size_t hv_shared_handle_size(void) { return sizeof(cudaIpcMemHandle_t); }

hv_status hv_shared_alloc(hv_context* ctx, size_t bytes, void** dev_ptr, uint8_t* handle) {
  return guarded([&] {
    require(ctx);
    if (!dev_ptr || !handle || bytes == 0) invalid("shared_alloc: bad arguments");
    ck(cudaMalloc(dev_ptr, bytes), "cudaMalloc");
    ck(cudaMemset(*dev_ptr, 0, bytes), "cudaMemset");
    cudaIpcMemHandle_t h;
    ck(cudaIpcGetMemHandle(&h, *dev_ptr), "cudaIpcGetMemHandle");
    std::memcpy(handle, &h, sizeof(h));
  });
}

hv_status hv_shared_open(hv_context* ctx, const uint8_t* handle, void** dev_ptr) {
  return guarded([&] {
    require(ctx);
    if (!dev_ptr || !handle) invalid("shared_open: bad arguments");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof(h));
    ck(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
  });
}

hv_status hv_shared_close(hv_context* ctx, void* dev_ptr) {
  return guarded([&] {
    require(ctx);
    ck(cudaIpcCloseMemHandle(dev_ptr), "cudaIpcCloseMemHandle");
  });
}

hv_status hv_shared_free(hv_context* ctx, void* dev_ptr) {
  return guarded([&] {
    require(ctx);
    ck(cudaFree(dev_ptr), "cudaFree");
  });
}

hv_status hv_dev_class_counts_peers_pitched(hv_context* ctx, const uint32_t* encoded, size_t ldw, size_t rows,
                                            size_t dim, const int32_t* labels, size_t class_count,
                                            uint32_t* const* peer_counts, uint64_t* const* peer_class_rows,
                                            size_t world) {
  return guarded([&] {
    require(ctx);
    if (class_count == 0) invalid("class_counts: need at least one class");
    if (world == 0 || world > 64) invalid("class_counts_peers: world must be 1..64");
    if (rows == 0) return;
    cudaStream_t st = ctx->stream;
    const size_t C = class_count, W = words_per_row(dim);
    DevBuf<uint32_t> hist(C, st), cursor(C, st), perm(rows, st);
    DevBuf<uint64_t> offsets(C + 1, st);
    hist.zero();
    label_bucket_device(ctx, st, labels, rows, C, hist.ptr, offsets.ptr, cursor.ptr, perm.ptr);
    launch_column_count_peers(st, encoded, static_cast<uint32_t>(W), perm.ptr, offsets.ptr, static_cast<uint32_t>(C),
                              rows, nullptr, peer_counts, static_cast<uint32_t>(world), static_cast<uint32_t>(ldw));
    add_rows_peers_kernel<<<grid_for(C * world, 128), 128, 0, st>>>(hist.ptr, static_cast<uint32_t>(C),
                                                                   peer_class_rows, static_cast<uint32_t>(world));
    launched("add_rows_peers_kernel");
  });
}

hv_status hv_dev_class_counts_peers(hv_context* ctx, const uint32_t* encoded, size_t rows, size_t dim,
                                    const int32_t* labels, size_t class_count, uint32_t* const* peer_counts,
                                    uint64_t* const* peer_class_rows, size_t world) {
  return hv_dev_class_counts_peers_pitched(ctx, encoded, 0, rows, dim, labels, class_count, peer_counts,
                                           peer_class_rows, world);
}

hv_status hv_dev_signal_peers(hv_context* ctx, uint32_t* const* peer_flags, size_t world, size_t rank,
                              uint32_t epoch) {
  return guarded([&] {
    require(ctx);
    if (rank >= world) invalid("signal_peers: rank >= world");
    signal_peers_kernel<<<1, 32, 0, ctx->stream>>>(peer_flags, static_cast<uint32_t>(world),
                                                   static_cast<uint32_t>(rank), epoch);
    launched("signal_peers_kernel");
  });
}

hv_status hv_dev_wait_peers(hv_context* ctx, const uint32_t* flags, size_t world, uint32_t epoch) {
  return guarded([&] {
    require(ctx);
    wait_peers_kernel<<<1, 32, 0, ctx->stream>>>(flags, static_cast<uint32_t>(world), epoch, ctx->d_err);
    launched("wait_peers_kernel");
  });
}

}  // extern "C"
