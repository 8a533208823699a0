// hv_stage.h — host thread pool and pinned staging of uint32 bin rows
// (hv_stage.cu).
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "hv_internal.cuh"

namespace hvb {

// Persistent workers for data-parallel host loops; the calling thread joins in.
class ThreadPool {
 public:
  explicit ThreadPool(unsigned workers);
  ~ThreadPool();
  ThreadPool(const ThreadPool&) = delete;
  ThreadPool& operator=(const ThreadPool&) = delete;
  void parallel_for(size_t n, const std::function<void(size_t)>& fn);
  unsigned size() const { return static_cast<unsigned>(workers_.size()); }

 private:
  void loop();
  void drain();
  std::vector<std::thread> workers_;
  std::mutex m_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(size_t)>* job_ = nullptr;
  size_t n_ = 0;
  std::atomic<size_t> next_{0}, left_{0};
  uint64_t gen_ = 0;
  bool stop_ = false;
};

// Pinned staging slots (ring of kSlots) + the pool that fills them.
struct HostStager {
  static constexpr int kSlots = 3;
  ThreadPool pool;
  uint8_t* slot[kSlots] = {};
  cudaEvent_t done[kSlots] = {};  // recorded after the slot's H2D copy
  size_t cap = 0;
  // streamed mode (encode_host_bins_streamed): copies run on their own stream
  // and each is followed by an 8-byte copy of the rows-landed count (pinned
  // flag[s], reused with slot s) into the encoder's `ready` word
  cudaStream_t copy = nullptr;
  unsigned long long* flag = nullptr;

  HostStager();
  ~HostStager();
  void reserve(size_t bytes);
  // Narrows rows x F uint32 bins into slot s (pitch ldb, zero padded);
  // returns the first flat index whose bin is >= B, or ~0.
  uint64_t narrow(const uint32_t* in, size_t rows, size_t F, size_t B, size_t ldb, int s);
};

unsigned host_thread_count();
// rows [r0, r1) of F uint32 bins -> uint8 rows of pitch ldb (zero padded), on
// the calling thread; returns the largest bin seen (hv_narrow.cpp).
uint32_t narrow_rows(const uint32_t* in, size_t F, size_t r0, size_t r1, uint8_t* out, size_t ldb);
// rows x F uint32 bins -> uint8 rows of pitch ldb (zero padded) on the pool;
// returns the first flat index whose bin is >= B, or ~0.
uint64_t narrow_rows_host(ThreadPool& pool, const uint32_t* in, size_t rows, size_t F, size_t B, uint8_t* out,
                          size_t ldb);
HostStager& stager(hv_context* ctx);
void destroy_stager(hv_context* ctx);
size_t stage_chunk_rows(size_t rows, size_t F);

// Host uint32 bin rows -> (narrow on host, pinned slot, H2D, encode) in chunks
// alternating the context's two streams. Chunk k (rows r0 .. r0+n) is encoded
// into out_for(r0, k) (row pitch ldo words, 0 = unpitched); b8 = two device chunk buffers of chunk * bins_pitch(F)
// bytes; `after(r0, n, k, stream)` runs per chunk (e.g. to enqueue a D2H of it
// on its stream). Returns the first offending flat bin index (relative to
// `bins`) or ~0; on an error the remaining chunks are not enqueued.
using ChunkOut = std::function<uint32_t*(size_t r0, size_t k)>;
using ChunkAfter = std::function<void(size_t r0, size_t n, size_t k, cudaStream_t st)>;
uint64_t encode_host_bins(hv_context* ctx, const uint32_t* bins, size_t rows, size_t F, size_t B, size_t D,
                          hv_binding binding, const uint32_t* d_id, const uint32_t* d_val, const uint32_t* d_tie,
                          const ChunkOut& out_for, DevBuf<uint8_t>* b8, size_t chunk, size_t& k,
                          const ChunkAfter& after = {}, size_t ldo = 0);

// Streamed variant for the table encoder: ONE persistent encoder launch on
// `kst` over all rows of d_bins (rows x bins_pitch(F), device, caller-owned,
// alive until kst has passed the launch) whose work items wait on *d_ready
// (rows landed so far); the host narrows chunks into the pinned slots and
// copies them (and the advancing row count) on the stager's copy stream.
// No per-chunk kernel boundaries (each cost a wave tail: 81 launches of 87 k
// rows 116.2 ms on two streams vs 113.8 ms in one launch). `launched` is set
// false, with nothing enqueued, when the table encoder does not apply (the
// caller then uses encode_host_bins). Returns the first bad flat bin index or
// ~0; on an error the launch is aborted (ready = ~0: work items not yet
// started are skipped) and its output is garbage.
uint64_t encode_host_bins_streamed(hv_context* ctx, const uint32_t* bins, size_t rows, size_t F, size_t B, size_t D,
                                   const uint32_t* d_id, const uint32_t* d_val, const uint32_t* d_tie,
                                   uint8_t* d_bins, uint32_t* out, size_t ldo, cudaStream_t kst,
                                   unsigned long long* d_ready, bool& launched);

// Copies `bytes` of (pageable) host memory to the device on the context
// stream through the pinned staging ring (host threads fill a slot while the
// previous one is in flight).
void upload_host(hv_context* ctx, const void* src, size_t bytes, void* dst);

}  // namespace hvb
