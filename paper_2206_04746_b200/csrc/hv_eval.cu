// hv_eval.cu — post-processing of concatenated fold predictions on device
// (eval.cpp:12-116): centred-majority label smoothing, sample confusion
// counts against one positive class, and episode (run-level) detection counts.
//
// All three are HBM-streaming integer passes over n int32 labels (4-8 B per
// sample read, 4 B written for smoothing); they run on the labels the
// prediction kernels left in HBM so an experiment never ships its predictions
// to the host before scoring. Results are bit-identical to the reference:
// integer counts, and ratios formed on the host with the reference's own
// double expressions (sample_metrics eval.cpp:66-75).
#include <cub/cub.cuh>

#include "hv_internal.cuh"

namespace hvb {
namespace {

constexpr unsigned kBlock = 256;

unsigned stream_grid(hv_context* ctx, size_t n) {
  return grid_for(n, kBlock, static_cast<unsigned>(ctx->sm_count) * 8u);
}

// --------------------------------------------------------------- smooth ----
// eval.cpp:18-24: the first non-binary label (lowest index) is the error.
__global__ void binary_check_kernel(const int32_t* __restrict__ labels, uint64_t n,
                                    unsigned long long* __restrict__ bad) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const int32_t v = labels[i];
    if (v != 0 && v != 1) atomicMin(bad, static_cast<unsigned long long>(i));
  }
}

// eval.cpp:25-36: prefix[i] = ones before i (prefix[n] = total);
// window [start, start + len) shifted inward at the edges, ties -> 1.
__global__ void smooth_kernel(const uint32_t* __restrict__ prefix, uint64_t n, uint64_t len, uint64_t half,
                              int32_t* __restrict__ out) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t start = i > half ? i - half : 0;
    start = start < n - len ? start : n - len;
    const uint64_t ones = prefix[start + len] - prefix[start];
    out[i] = 2 * ones >= len ? 1 : 0;
  }
}

struct ToU32 {
  __device__ __forceinline__ uint32_t operator()(int32_t v) const { return static_cast<uint32_t>(v); }
};

// ------------------------------------------------------------- confusion ----
// eval.cpp:52-65: tp / fp / tn / fn against positive_class and exact matches.
__global__ void confusion_kernel(const int32_t* __restrict__ pred, const int32_t* __restrict__ truth, uint64_t n,
                                 int positive, unsigned long long* __restrict__ out) {
  unsigned long long c[5] = {0, 0, 0, 0, 0};
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const int32_t p = pred[i], t = truth[i];
    c[4] += p == t;
    const bool pp = p == positive, tt = t == positive;
    c[0] += pp && tt;
    c[1] += pp && !tt;
    c[3] += !pp && tt;
    c[2] += !pp && !tt;
  }
  using Reduce = cub::BlockReduce<unsigned long long, kBlock>;
  __shared__ typename Reduce::TempStorage tmp;
#pragma unroll
  for (int k = 0; k < 5; ++k) {
    const unsigned long long s = Reduce(tmp).Sum(c[k]);
    if (threadIdx.x == 0 && s) atomicAdd(out + k, s);
    __syncthreads();
  }
}

// -------------------------------------------------------------- episodes ----
// eval.cpp:79-116 as one scan. Per sample: hits of the truth-run kind
// (truth and pred positive) and of the prediction-run kind (the same
// samples: a prediction run "overlaps" truth exactly where a hit lies),
// plus the index of the latest run start of each kind (max-scan).
// A run ending at e with start s is detected / overlapping iff
// hits[e] - hits[s - 1] > 0 (inclusive prefix).
struct EpisodeScan {
  uint32_t hits;
  int32_t truth_start;
  int32_t pred_start;
};

struct EpisodeOp {
  __device__ __forceinline__ EpisodeScan operator()(const EpisodeScan& a, const EpisodeScan& b) const {
    return {a.hits + b.hits, a.truth_start > b.truth_start ? a.truth_start : b.truth_start,
            a.pred_start > b.pred_start ? a.pred_start : b.pred_start};
  }
};

struct EpisodeInput {
  const int32_t* pred;
  const int32_t* truth;
  int positive;
  __device__ __forceinline__ EpisodeScan operator()(int64_t i) const {
    const bool t = truth[i] == positive, p = pred[i] == positive;
    const bool t0 = i > 0 && truth[i - 1] == positive, p0 = i > 0 && pred[i - 1] == positive;
    return {static_cast<uint32_t>(t && p), t && !t0 ? static_cast<int32_t>(i) : -1,
            p && !p0 ? static_cast<int32_t>(i) : -1};
  }
};

__global__ void episode_count_kernel(const int32_t* __restrict__ pred, const int32_t* __restrict__ truth, uint64_t n,
                                     int positive, const EpisodeScan* __restrict__ scan,
                                     unsigned long long* __restrict__ out) {
  unsigned long long c[3] = {0, 0, 0};  // detected, total, false_positive
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const bool t = truth[i] == positive, p = pred[i] == positive;
    const bool t1 = i + 1 < n && truth[i + 1] == positive, p1 = i + 1 < n && pred[i + 1] == positive;
    const EpisodeScan e = scan[i];
    if (t && !t1) {  // truth run ends here
      const int32_t s = e.truth_start;
      const uint32_t before = s > 0 ? scan[s - 1].hits : 0u;
      c[1] += 1;
      c[0] += e.hits > before;
    }
    if (p && !p1) {  // prediction run ends here
      const int32_t s = e.pred_start;
      const uint32_t before = s > 0 ? scan[s - 1].hits : 0u;
      c[2] += e.hits == before;
    }
  }
  using Reduce = cub::BlockReduce<unsigned long long, kBlock>;
  __shared__ typename Reduce::TempStorage tmp;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const unsigned long long s = Reduce(tmp).Sum(c[k]);
    if (threadIdx.x == 0 && s) atomicAdd(out + k, s);
    __syncthreads();
  }
}

// ------------------------------------------------------------ compaction ----
struct Tested {
  const int32_t* predicted;
  __device__ __forceinline__ bool operator()(uint64_t i) const { return predicted[i] >= 0; }
};

__global__ void gather_sequences_kernel(const uint64_t* __restrict__ tested, uint64_t m,
                                        const int32_t* __restrict__ predicted, const int32_t* __restrict__ y,
                                        int32_t* __restrict__ pred_seq, int32_t* __restrict__ truth_seq) {
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < m; k += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i = tested[k];
    pred_seq[k] = predicted[i];
    truth_seq[k] = y[i];
  }
}

__global__ void scatter_labels_kernel(const uint64_t* __restrict__ idx, uint64_t n, const int32_t* __restrict__ lab,
                                      int32_t* __restrict__ predicted) {
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < n; k += (uint64_t)gridDim.x * blockDim.x) {
    predicted[idx[k]] = lab[k];
  }
}

}  // namespace

void smooth_labels_device(hv_context* ctx, cudaStream_t st, const int32_t* labels, size_t n, size_t window,
                          int32_t* out) {
  if (window == 0 || window % 2 == 0) {
    invalid("smooth_labels: window must be odd and >= 1, got " + std::to_string(window));
  }
  if (n > 0xFFFFFFFFull) invalid("smooth_labels: more than 2^32 labels");
  if (n == 0) return;
  DevBuf<unsigned long long> bad(1, st);
  ck(cudaMemsetAsync(bad.ptr, 0xFF, sizeof(unsigned long long), st), "memset");
  binary_check_kernel<<<stream_grid(ctx, n), kBlock, 0, st>>>(labels, n, bad.ptr);
  launched("binary_check_kernel");
  unsigned long long first_bad = ~0ull;
  ck(cudaMemcpyAsync(&first_bad, bad.ptr, sizeof(first_bad), cudaMemcpyDeviceToHost, st), "D2H");
  ck(cudaStreamSynchronize(st), "cudaStreamSynchronize");
  if (first_bad != ~0ull) {
    int32_t v = 0;
    ck(cudaMemcpy(&v, labels + first_bad, sizeof(v), cudaMemcpyDeviceToHost), "D2H label");
    invalid("smooth_labels: non-binary label " + std::to_string(v) + " at index " + std::to_string(first_bad));
  }
  if (window == 1) {
    if (out != labels) ck(cudaMemcpyAsync(out, labels, n * sizeof(int32_t), cudaMemcpyDeviceToDevice, st), "D2D");
    return;
  }
  // prefix[0] = 0, prefix[i + 1] = ones in labels[0..i]
  DevBuf<uint32_t> prefix(n + 1, st);
  ck(cudaMemsetAsync(prefix.ptr, 0, sizeof(uint32_t), st), "memset");
  cub::TransformInputIterator<uint32_t, ToU32, const int32_t*> in(labels, ToU32{});
  size_t tmp_bytes = 0;
  ck(cub::DeviceScan::InclusiveSum(nullptr, tmp_bytes, in, prefix.ptr + 1, static_cast<int64_t>(n), st), "scan size");
  DevBuf<uint8_t> tmp(tmp_bytes, st);
  ck(cub::DeviceScan::InclusiveSum(tmp.ptr, tmp_bytes, in, prefix.ptr + 1, static_cast<int64_t>(n), st), "scan");
  launched("cub::DeviceScan (smooth prefix)");
  const uint64_t len = window < n ? window : n;
  smooth_kernel<<<stream_grid(ctx, n), kBlock, 0, st>>>(prefix.ptr, n, len, (window - 1) / 2, out);
  launched("smooth_kernel");
}

void confusion_device(hv_context* ctx, cudaStream_t st, const int32_t* pred, const int32_t* truth, size_t n,
                      int positive, unsigned long long* out5) {
  ck(cudaMemsetAsync(out5, 0, 5 * sizeof(unsigned long long), st), "memset");
  if (n == 0) return;
  confusion_kernel<<<stream_grid(ctx, n), kBlock, 0, st>>>(pred, truth, n, positive, out5);
  launched("confusion_kernel");
}

void episodes_device(hv_context* ctx, cudaStream_t st, const int32_t* pred, const int32_t* truth, size_t n,
                     int positive, unsigned long long* out3) {
  ck(cudaMemsetAsync(out3, 0, 3 * sizeof(unsigned long long), st), "memset");
  if (n == 0) return;
  if (n > 0x7FFFFFFFull) invalid("episode_metrics: more than 2^31 labels");
  DevBuf<EpisodeScan> scan(n, st);
  cub::CountingInputIterator<int64_t> idx(0);
  cub::TransformInputIterator<EpisodeScan, EpisodeInput, cub::CountingInputIterator<int64_t>> in(
      idx, EpisodeInput{pred, truth, positive});
  size_t tmp_bytes = 0;
  ck(cub::DeviceScan::InclusiveScan(nullptr, tmp_bytes, in, scan.ptr, EpisodeOp{}, static_cast<int64_t>(n), st),
     "scan size");
  DevBuf<uint8_t> tmp(tmp_bytes, st);
  ck(cub::DeviceScan::InclusiveScan(tmp.ptr, tmp_bytes, in, scan.ptr, EpisodeOp{}, static_cast<int64_t>(n), st),
     "scan");
  launched("cub::DeviceScan (episode runs)");
  episode_count_kernel<<<stream_grid(ctx, n), kBlock, 0, st>>>(pred, truth, n, positive, scan.ptr, out3);
  launched("episode_count_kernel");
}

// eval.cpp:66-75 on the host from exact integer counts.
void fill_report(const unsigned long long c5[5], const unsigned long long e3[3], size_t n, hv_eval_report* r) {
  r->tp = c5[0];
  r->fp = c5[1];
  r->tn = c5[2];
  r->fn = c5[3];
  r->accuracy = static_cast<double>(c5[4]) / static_cast<double>(n);
  r->has_tpr = r->tp + r->fn > 0;
  r->has_ppv = r->tp + r->fp > 0;
  r->tpr = r->has_tpr ? static_cast<double>(r->tp) / static_cast<double>(r->tp + r->fn) : __builtin_nan("");
  r->ppv = r->has_ppv ? static_cast<double>(r->tp) / static_cast<double>(r->tp + r->fp) : __builtin_nan("");
  r->has_f1 = r->has_tpr && r->has_ppv && (r->tpr + r->ppv) > 0.0;
  r->f1 = r->has_f1 ? 2.0 * r->ppv * r->tpr / (r->ppv + r->tpr) : __builtin_nan("");
  r->episodes_detected = e3 ? e3[0] : 0;
  r->episodes_total = e3 ? e3[1] : 0;
  r->episodes_false_positive = e3 ? e3[2] : 0;
}

void scatter_labels_device(hv_context* ctx, cudaStream_t st, const uint64_t* idx, size_t n, const int32_t* lab,
                           int32_t* predicted) {
  if (n == 0) return;
  scatter_labels_kernel<<<stream_grid(ctx, n), kBlock, 0, st>>>(idx, n, lab, predicted);
  launched("scatter_labels_kernel");
}

// experiment.cpp:314-330: tested rows in original order and their pred/truth.
size_t compact_tested_device(hv_context* ctx, cudaStream_t st, const int32_t* predicted, const int32_t* y,
                             size_t rows, DevBuf<uint64_t>& tested, DevBuf<int32_t>& pred_seq,
                             DevBuf<int32_t>& truth_seq) {
  tested = DevBuf<uint64_t>(std::max<size_t>(rows, 1), st);
  DevBuf<uint64_t> count(1, st);
  cub::CountingInputIterator<uint64_t> it(0);
  size_t tmp_bytes = 0;
  ck(cub::DeviceSelect::If(nullptr, tmp_bytes, it, tested.ptr, count.ptr, static_cast<int64_t>(rows),
                           Tested{predicted}, st),
     "select size");
  DevBuf<uint8_t> tmp(tmp_bytes, st);
  ck(cub::DeviceSelect::If(tmp.ptr, tmp_bytes, it, tested.ptr, count.ptr, static_cast<int64_t>(rows),
                           Tested{predicted}, st),
     "select");
  launched("cub::DeviceSelect (tested rows)");
  uint64_t m = 0;
  ck(cudaMemcpyAsync(&m, count.ptr, sizeof(m), cudaMemcpyDeviceToHost, st), "D2H");
  ck(cudaStreamSynchronize(st), "cudaStreamSynchronize");
  pred_seq = DevBuf<int32_t>(std::max<uint64_t>(m, 1), st);
  truth_seq = DevBuf<int32_t>(std::max<uint64_t>(m, 1), st);
  if (m) {
    gather_sequences_kernel<<<stream_grid(ctx, m), kBlock, 0, st>>>(tested.ptr, m, predicted, y, pred_seq.ptr,
                                                                    truth_seq.ptr);
    launched("gather_sequences_kernel");
  }
  return m;
}

}  // namespace hvb

using namespace hvb;

extern "C" {

hv_status hv_dev_smooth_labels(hv_context* ctx, const int32_t* labels, size_t n, size_t window, int32_t* out) {
  return guarded([&] {
    require(ctx);
    smooth_labels_device(ctx, ctx->stream, labels, n, window, out);
  });
}

hv_status hv_dev_eval_counts(hv_context* ctx, const int32_t* pred, const int32_t* truth, size_t n,
                             int positive_class, uint64_t* confusion5, uint64_t* episodes3) {
  return guarded([&] {
    require(ctx);
    if (confusion5) {
      confusion_device(ctx, ctx->stream, pred, truth, n, positive_class,
                       reinterpret_cast<unsigned long long*>(confusion5));
    }
    if (episodes3) {
      episodes_device(ctx, ctx->stream, pred, truth, n, positive_class,
                      reinterpret_cast<unsigned long long*>(episodes3));
    }
  });
}

hv_status hv_smooth_labels(hv_context* ctx, const int32_t* labels, size_t n, size_t window, int32_t* out) {
  return guarded([&] {
    require(ctx);
    cudaStream_t st = ctx->stream;
    if (window == 0 || window % 2 == 0) {
      invalid("smooth_labels: window must be odd and >= 1, got " + std::to_string(window));
    }
    if (n == 0) return;
    DevBuf<int32_t> in(n, st), out_d(n, st);
    in.upload(labels);
    smooth_labels_device(ctx, st, in.ptr, n, window, out_d.ptr);
    out_d.download(out);
    sync(ctx);
  });
}

hv_status hv_sample_metrics(hv_context* ctx, const int32_t* pred, size_t n_pred, const int32_t* truth,
                            size_t n_truth, int positive_class, hv_eval_report* report) {
  return guarded([&] {
    require(ctx);
    if (n_pred != n_truth) {
      invalid("sample_metrics: " + std::to_string(n_pred) + " predictions vs " + std::to_string(n_truth) +
              " labels");
    }
    if (n_pred == 0) invalid("sample_metrics: empty sequences");
    if (!report) invalid("sample_metrics: null report");
    cudaStream_t st = ctx->stream;
    DevBuf<int32_t> p(n_pred, st), t(n_pred, st);
    p.upload(pred);
    t.upload(truth);
    DevBuf<unsigned long long> c(5, st);
    confusion_device(ctx, st, p.ptr, t.ptr, n_pred, positive_class, c.ptr);
    unsigned long long h[5];
    c.download(h);
    sync(ctx);
    fill_report(h, nullptr, n_pred, report);
  });
}

hv_status hv_episode_metrics(hv_context* ctx, const int32_t* pred, size_t n_pred, const int32_t* truth,
                             size_t n_truth, int positive_class, uint64_t* detected, uint64_t* total,
                             uint64_t* false_positive) {
  return guarded([&] {
    require(ctx);
    if (n_pred != n_truth) {
      invalid("episode_metrics: " + std::to_string(n_pred) + " predictions vs " + std::to_string(n_truth) +
              " labels");
    }
    cudaStream_t st = ctx->stream;
    unsigned long long h[3] = {0, 0, 0};
    if (n_pred) {
      DevBuf<int32_t> p(n_pred, st), t(n_pred, st);
      p.upload(pred);
      t.upload(truth);
      DevBuf<unsigned long long> e(3, st);
      episodes_device(ctx, st, p.ptr, t.ptr, n_pred, positive_class, e.ptr);
      e.download(h);
      sync(ctx);
    }
    if (detected) *detected = h[0];
    if (total) *total = h[1];
    if (false_positive) *false_positive = h[2];
  });
}

}  // extern "C"
