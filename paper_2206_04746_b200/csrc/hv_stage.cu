// hv_stage.cu — host-side staging of the reference's uint32 bin rows.
//
// The reference API hands encode_batch / run_fold_packed a row-major
// std::vector<uint32_t> of bin indices (encoding.hpp:85-93, experiment.cpp:
// 159-166): 4 bytes per feature, usually pageable. Copying that verbatim is
// PCIe-bound (1,368 B/row at CHB-MIT: 55 GB/s pinned, 11 GB/s pageable on the
// B200 host). Instead the host threads of the context narrow each chunk to the
// device's uint8 layout (row pitch bins_pitch(F), zero padding) directly into a
// pinned staging slot, validating every bin against B on the way (encoding.cpp
// :43-55), and the slot is DMA'd while the next chunk is narrowed and the
// previous one encoded:
//
//   host:   narrow k+1 ──────────────── narrow k+2 ───
//   copy:        H2D k ────── H2D k+1 ────
//   SMs:              encode k ───────── encode k+1 ───
//
// 3.6x fewer PCIe bytes, and pageable inputs cost the same as pinned ones.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <condition_variable>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "hv_internal.cuh"
#include "hv_stage.h"

namespace hvb {

// ---------------------------------------------------------- thread pool ----
ThreadPool::ThreadPool(unsigned n) {
  for (unsigned i = 0; i < n; ++i) workers_.emplace_back([this] { loop(); });
}

ThreadPool::~ThreadPool() {
  {
    std::lock_guard<std::mutex> g(m_);
    stop_ = true;
  }
  cv_.notify_all();
  for (auto& t : workers_) t.join();
}

void ThreadPool::loop() {
  uint64_t seen = 0;
  for (;;) {
    {
      std::unique_lock<std::mutex> g(m_);
      cv_.wait(g, [&] { return stop_ || gen_ != seen; });
      if (stop_) return;
      seen = gen_;
    }
    drain();
  }
}

void ThreadPool::drain() {
  for (;;) {
    const size_t i = next_.fetch_add(1, std::memory_order_relaxed);
    if (i >= n_) break;
    (*job_)(i);
    if (left_.fetch_sub(1, std::memory_order_acq_rel) == 1) {
      std::lock_guard<std::mutex> g(m_);
      done_cv_.notify_all();
    }
  }
}

void ThreadPool::parallel_for(size_t n, const std::function<void(size_t)>& fn) {
  if (n == 0) return;
  {
    std::lock_guard<std::mutex> g(m_);
    job_ = &fn;
    n_ = n;
    next_.store(0);
    left_.store(n);
    ++gen_;
  }
  cv_.notify_all();
  drain();  // the caller works too
  std::unique_lock<std::mutex> g(m_);
  done_cv_.wait(g, [&] { return left_.load() == 0; });
  job_ = nullptr;
}

unsigned host_thread_count() {
  if (const char* e = getenv("HVB200_HOST_THREADS")) {
    const int n = atoi(e);
    if (n >= 1) return static_cast<unsigned>(n);
  }
  unsigned hc = std::thread::hardware_concurrency();
  hc = hc ? hc : 1u;
  // one process per GPU (torchrun sets LOCAL_WORLD_SIZE): share the host cores
  if (const char* lw = getenv("LOCAL_WORLD_SIZE")) {
    const int n = atoi(lw);
    if (n > 1) hc = std::max(1u, hc / static_cast<unsigned>(n));
  }
  return std::max(1u, std::min(hc, 64u));
}

HostStager::HostStager() : pool(host_thread_count() - 1) {
  for (int i = 0; i < kSlots; ++i) {
    ck(cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming), "cudaEventCreate");
  }
  ck(cudaStreamCreateWithFlags(&copy, cudaStreamNonBlocking), "cudaStreamCreate");
  ck(cudaHostAlloc(reinterpret_cast<void**>(&flag), kSlots * sizeof(unsigned long long), cudaHostAllocDefault),
     "cudaHostAlloc");
}

HostStager::~HostStager() {
  for (int i = 0; i < kSlots; ++i) {
    if (done[i]) {
      cudaEventSynchronize(done[i]);
      cudaEventDestroy(done[i]);
    }
    if (slot[i]) cudaFreeHost(slot[i]);
  }
  if (copy) {
    cudaStreamSynchronize(copy);
    cudaStreamDestroy(copy);
  }
  if (flag) cudaFreeHost(flag);
}

void HostStager::reserve(size_t bytes) {
  if (bytes <= cap) return;
  for (int i = 0; i < kSlots; ++i) {
    if (slot[i]) {
      ck(cudaEventSynchronize(done[i]), "cudaEventSynchronize");
      ck(cudaFreeHost(slot[i]), "cudaFreeHost");
      slot[i] = nullptr;
    }
  }
  cap = 0;
  for (int i = 0; i < kSlots; ++i) ck(cudaHostAlloc(&slot[i], bytes, cudaHostAllocDefault), "cudaHostAlloc");
  cap = bytes;
}

uint64_t narrow_rows_host(ThreadPool& pool, const uint32_t* in, size_t rows, size_t F, size_t B, uint8_t* out,
                          size_t ldb) {
  if (rows == 0) return ~0ull;
  const unsigned parts = std::max<unsigned>(1, (pool.size() + 1) * 4);
  const size_t per = (rows + parts - 1) / parts;
  const size_t pieces = (rows + per - 1) / per;
  std::vector<uint32_t> mx(pieces, 0);
  pool.parallel_for(pieces, [&](size_t i) {
    const size_t r0 = i * per, r1 = std::min(rows, r0 + per);
    mx[i] = narrow_rows(in, F, r0, r1, out, ldb);
  });
  for (size_t i = 0; i < pieces; ++i) {
    if (mx[i] >= B) {  // error path: first offending flat index in this piece
      const size_t r0 = i * per, r1 = std::min(rows, r0 + per);
      for (size_t k = r0 * F; k < r1 * F; ++k) {
        if (in[k] >= B) return k;
      }
    }
  }
  return ~0ull;
}

uint64_t HostStager::narrow(const uint32_t* in, size_t rows, size_t F, size_t B, size_t ldb, int s) {
  return narrow_rows_host(pool, in, rows, F, B, slot[s], ldb);
}

HostStager& stager(hv_context* ctx) {
  if (!ctx->stager) ctx->stager = new HostStager();
  return *ctx->stager;
}

void destroy_stager(hv_context* ctx) {
  delete ctx->stager;
  ctx->stager = nullptr;
}

size_t stage_chunk_rows(size_t rows, size_t F) {
  // ~32 MB of uint8 per slot (a chunk is still several encoder waves): the
  // e2e CHB-MIT fold measured 54.8 M dp/s at 32 MB vs 53.7 M at 96 MB and
  // 48.0 M at 384 MB (shorter head and tail of the pipeline)
  const size_t ldb = bins_pitch(F);
  size_t mb = 32;
  if (const char* e = getenv("HVB200_STAGE_MB")) mb = std::max<size_t>(1, static_cast<size_t>(atoll(e)));  // tuning
  return std::max<size_t>(1, std::min<size_t>(std::max<size_t>(rows, 1), (mb << 20) / ldb));
}

uint64_t encode_host_bins(hv_context* ctx, const uint32_t* bins, size_t rows, size_t F, size_t B, size_t D,
                          hv_binding binding, const uint32_t* d_id, const uint32_t* d_val, const uint32_t* d_tie,
                          const ChunkOut& out_for, DevBuf<uint8_t>* b8, size_t chunk, size_t& k,
                          const ChunkAfter& after, size_t ldo) {
  check_bins_u8(B, "encode");
  const size_t ldb = bins_pitch(F);
  HostStager& hs = stager(ctx);
  hs.reserve(chunk * ldb);
  cudaStream_t streams[2] = {ctx->stream, ctx->aux};
  // HVB200_STAGE_PROFILE=1: host time spent waiting for a free slot vs narrowing
  static const bool prof = getenv("HVB200_STAGE_PROFILE") != nullptr;
  using clk = std::chrono::steady_clock;
  const auto t_call = clk::now();
  double wait_ms = 0, narrow_ms = 0;
  size_t pieces = 0;
  // the first chunks of a call ramp up (1/8, 1/4, 1/2 of a slot) so the SMs
  // start encoding after a short narrow + copy instead of a full slot's
  size_t step = k == 0 ? std::max<size_t>(1, chunk / 8) : chunk;
  const size_t tail_min = std::max<size_t>(1, chunk / 16);
  for (size_t r0 = 0, n = 0; r0 < rows; r0 += n, ++k, step = std::min(chunk, 2 * step)) {
    n = std::min(step, rows - r0);
    // ... and ramp down over the last two slots (halving pieces), so the
    // encode left after the final copy is a short one
    const size_t left = rows - r0;
    if (left <= 2 * step && left > tail_min) n = std::max(tail_min, (left + 1) / 2);
    const int s = static_cast<int>(k % HostStager::kSlots);
    cudaStream_t st = streams[k & 1];
    const auto t0 = clk::now();
    ck(cudaEventSynchronize(hs.done[s]), "stage slot wait");  // its previous H2D has finished
    const auto t1 = clk::now();
    const uint64_t bad = hs.narrow(bins + r0 * F, n, F, B, ldb, s);
    if (prof) {
      wait_ms += std::chrono::duration<double, std::milli>(t1 - t0).count();
      narrow_ms += std::chrono::duration<double, std::milli>(clk::now() - t1).count();
      ++pieces;
    }
    if (bad != ~0ull) return r0 * F + bad;
    ck(cudaMemcpyAsync(b8[k & 1].ptr, hs.slot[s], n * ldb, cudaMemcpyHostToDevice, st), "H2D bins");
    ck(cudaEventRecord(hs.done[s], st), "cudaEventRecord");
    if (ldo == 0 || ldo == words_per_row(D)) {
      encode_device(ctx, st, b8[k & 1].ptr, ldb, n, F, d_id, d_val, B, D, binding, d_tie, out_for(r0, k));
    } else {
      encode_device(ctx, st, b8[k & 1].ptr, ldb, n, F, d_id, d_val, B, D, binding, d_tie, out_for(r0, k), true, 0,
                    words_per_row(D), ldo);
    }
    if (after) after(r0, n, k, st);
  }
  if (prof) {
    fprintf(stderr, "[stage] rows %zu pieces %zu chunk %zu threads %zu: host %.2f ms (slot wait %.2f, narrow %.2f)\n",
            rows, pieces, chunk, hs.pool.size() + 1,
            std::chrono::duration<double, std::milli>(clk::now() - t_call).count(), wait_ms, narrow_ms);
  }
  return ~0ull;
}

uint64_t encode_host_bins_streamed(hv_context* ctx, const uint32_t* bins, size_t rows, size_t F, size_t B, size_t D,
                                   const uint32_t* d_id, const uint32_t* d_val, const uint32_t* d_tie,
                                   uint8_t* d_bins, uint32_t* out, size_t ldo, cudaStream_t kst,
                                   unsigned long long* d_ready, bool& launched) {
  check_bins_u8(B, "encode");
  launched = false;
  if (rows == 0) {
    launched = true;
    return ~0ull;
  }
  const size_t ldb = bins_pitch(F), W = words_per_row(D);
  if (D > 0xFFFFFFFFull || F > 0xFFFFFFFFull) invalid("encode: shape too large");
  HostStager& hs = stager(ctx);
  const size_t chunk = stage_chunk_rows(rows, F);
  hs.reserve(chunk * ldb);
  ck(cudaMemsetAsync(d_ready, 0, sizeof(unsigned long long), kst), "ready reset");
  // the copies (and their ready updates) land after the reset — and must not
  // wait for the launch itself, which waits for them
  cudaEvent_t ev;
  ck(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "event");
  ck(cudaEventRecord(ev, kst), "event");
  ck(cudaStreamWaitEvent(hs.copy, ev, 0), "wait");
  cudaEventDestroy(ev);
  if (!launch_tt(ctx, kst, d_bins, static_cast<uint32_t>(ldb), rows, static_cast<uint32_t>(F), d_id, d_val,
                 static_cast<uint32_t>(B), static_cast<uint32_t>(D), static_cast<uint32_t>(W), d_tie, out, 0u,
                 static_cast<uint32_t>(W), static_cast<uint32_t>(ldo ? ldo : W), false, d_ready)) {
    return ~0ull;  // nothing launched (the reset alone is harmless)
  }
  launched = true;
  static const bool prof = getenv("HVB200_STAGE_PROFILE") != nullptr;
  using clk = std::chrono::steady_clock;
  const auto t_call = clk::now();
  double wait_ms = 0, narrow_ms = 0;
  size_t pieces = 0;
  // publishes rows [0, n) as landed, from slot s's pinned flag word
  auto publish = [&](unsigned long long n, int s) {
    hs.flag[s] = n;
    ck(cudaMemcpyAsync(d_ready, &hs.flag[s], sizeof(unsigned long long), cudaMemcpyHostToDevice, hs.copy),
       "H2D ready");
  };
  uint64_t bad = ~0ull;
  size_t k = 0;
  try {
    // ramp up (1/16, 1/8, ... of a slot): the first 16 k-row work block can
    // start after a short narrow + copy
    size_t step = std::max<size_t>(1, chunk / 16);
    for (size_t r0 = 0, n = 0; r0 < rows; r0 += n, ++k, step = std::min(chunk, 2 * step)) {
      n = std::min(step, rows - r0);
      const int s = static_cast<int>(k % HostStager::kSlots);
      const auto t0 = clk::now();
      ck(cudaEventSynchronize(hs.done[s]), "stage slot wait");  // slot s (and flag[s]) copied out
      const auto t1 = clk::now();
      bad = hs.narrow(bins + r0 * F, n, F, B, ldb, s);
      if (prof) {
        wait_ms += std::chrono::duration<double, std::milli>(t1 - t0).count();
        narrow_ms += std::chrono::duration<double, std::milli>(clk::now() - t1).count();
        ++pieces;
      }
      if (bad != ~0ull) {
        bad += r0 * F;
        publish(~0ull, s);  // abort the launch (its output is discarded by the caller)
        ck(cudaEventRecord(hs.done[s], hs.copy), "cudaEventRecord");
        return bad;
      }
      ck(cudaMemcpyAsync(d_bins + r0 * ldb, hs.slot[s], n * ldb, cudaMemcpyHostToDevice, hs.copy), "H2D bins");
      publish(r0 + n, s);
      ck(cudaEventRecord(hs.done[s], hs.copy), "cudaEventRecord");
    }
  } catch (...) {
    // never leave the launch spinning on rows that will not come
    // (on the non-blocking copy stream: a legacy-stream copy could queue
    // behind the launch itself)
    const unsigned long long abort_all = ~0ull;
    cudaMemcpyAsync(d_ready, &abort_all, sizeof(abort_all), cudaMemcpyHostToDevice, hs.copy);
    cudaStreamSynchronize(hs.copy);
    throw;
  }
  if (prof) {
    fprintf(stderr, "[stage] streamed rows %zu pieces %zu chunk %zu threads %zu: host %.2f ms (slot wait %.2f, "
            "narrow %.2f)\n", rows, pieces, chunk, hs.pool.size() + 1,
            std::chrono::duration<double, std::milli>(clk::now() - t_call).count(), wait_ms, narrow_ms);
  }
  return bad;
}

void upload_host(hv_context* ctx, const void* src, size_t bytes, void* dst) {
  if (bytes == 0) return;
  HostStager& hs = stager(ctx);
  const size_t chunk = std::min<size_t>(bytes, size_t(64) << 20);
  hs.reserve(chunk);
  const uint8_t* in = static_cast<const uint8_t*>(src);
  uint8_t* out = static_cast<uint8_t*>(dst);
  size_t k = 0;
  for (size_t off = 0; off < bytes; off += chunk, ++k) {
    const size_t n = std::min(chunk, bytes - off);
    const int slot = static_cast<int>(k % HostStager::kSlots);
    ck(cudaEventSynchronize(hs.done[slot]), "stage slot wait");
    const size_t parts = (hs.pool.size() + 1) * 2, per = (n + parts - 1) / parts;
    hs.pool.parallel_for((n + per - 1) / per, [&](size_t i) {
      const size_t a = i * per, b = std::min(n, a + per);
      std::memcpy(hs.slot[slot] + a, in + off + a, b - a);
    });
    ck(cudaMemcpyAsync(out + off, hs.slot[slot], n, cudaMemcpyHostToDevice, ctx->stream), "H2D upload");
    ck(cudaEventRecord(hs.done[slot], ctx->stream), "cudaEventRecord");
  }
}

}  // namespace hvb

extern "C" {

// Host-only narrowing (no device, no context): the staging kernel of the host
// pipeline, exposed for callers that stage bins themselves and for CPU tests.
hv_status hv_host_narrow_bins(const uint32_t* bins32, size_t rows, size_t features, size_t bins, uint8_t* out,
                              size_t ldb, uint64_t* first_bad) {
  return hvb::guarded([&] {
    if (ldb < features) hvb::invalid("narrow_bins: ldb must be >= features");
    if (bins > 256) hvb::invalid("narrow_bins: bins must be <= 256");
    static hvb::ThreadPool pool(hvb::host_thread_count() - 1);
    const uint64_t bad = hvb::narrow_rows_host(pool, bins32, rows, features, bins, out, ldb);
    if (first_bad) *first_bad = bad;
  });
}

}  // extern "C"
