// hypervec_gpu.cpp — drop-in replacement of the reference's hot-path functions.
//
// Compiled against the reference's own headers (-I /root/reference/proj/include)
// it defines the hypervec:: functions of kernels.hpp, encoding.hpp and
// model.hpp that carry the hot path (and the eval.hpp scoring of their
// predictions), each as a thin adapter over the C ABI of
// libhvb200 (include/hvb200.h): same signatures, same exceptions and messages.
// Linking this object ahead of the reference library (whose definitions of the
// same symbols are weakened, see dropin/Makefile) makes every existing caller —
// run_fold_packed, run_bench, the CLI, the acceptance gate — run on the B200
// without source changes. Codebook generation, I/O, data and experiment code
// stay the reference's.

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "hvb200.h"
#include "hypervec/bitmat.hpp"
#include "hypervec/encoding.hpp"
#include "hypervec/eval.hpp"
#include "hypervec/kernels.hpp"
#include "hypervec/model.hpp"

namespace {

hv_context* ctx() {
  static hv_context* c = [] {
    hv_context* h = nullptr;
    if (hv_context_create(0, &h) != HV_OK) throw std::runtime_error(hv_last_error());
    return h;
  }();
  return c;
}

void check(hv_status s) {
  if (s == HV_OK) return;
  const std::string msg = hv_last_error();
  switch (s) {
    case HV_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case HV_ERR_DOMAIN: throw std::domain_error(msg);
    case HV_ERR_LOGIC: throw std::logic_error(msg);
    default: throw std::runtime_error(msg);
  }
}

const uint32_t* W(const hypervec::PackedBitMatrix& m) { return m.words().data(); }
uint32_t* W(hypervec::PackedBitMatrix& m) { return m.words().data(); }

hv_model view(hypervec::HDModel& m) {
  return hv_model{m.config.class_count,
                  m.config.dim,
                  m.config.metric == hypervec::Metric::kHamming ? HV_METRIC_HAMMING : HV_METRIC_COSINE,
                  m.config.gamma,
                  m.config.seed,
                  m.accumulators.data(),
                  m.class_weight.data(),
                  m.sample_counts.data(),
                  W(m.class_vectors),
                  W(m.tiebreak)};
}

// HDModel storage for config (sizes follow make_empty_model, model.cpp:198-217)
hypervec::HDModel allocate(const hypervec::ModelConfig& cfg) {
  hypervec::HDModel m;
  m.config = cfg;
  m.accumulators.assign(cfg.class_count * cfg.dim, 0.0);
  m.class_weight.assign(cfg.class_count, 0.0);
  m.sample_counts.assign(cfg.class_count, 0);
  m.class_vectors = hypervec::PackedBitMatrix(cfg.class_count, cfg.dim);
  m.tiebreak = hypervec::PackedBitMatrix(1, cfg.dim);
  return m;
}

}  // namespace

namespace hypervec {

// ---------------------------------------------------------- kernels.hpp ----
PackedBitMatrix pack(const DenseBitMatrix& bits) {
  PackedBitMatrix out(bits.rows(), bits.dim());
  check(hv_pack(ctx(), bits.bits().data(), bits.rows(), bits.dim(), W(out)));
  return out;
}

DenseBitMatrix unpack(const PackedBitMatrix& m) {
  DenseBitMatrix out(m.rows(), m.dim());
  check(hv_unpack(ctx(), W(m), m.rows(), m.dim(), out.bits().data()));
  return out;
}

PackedBitMatrix xor_bind(const PackedBitMatrix& a, const PackedBitMatrix& b) {
  PackedBitMatrix out(a.rows(), a.dim());
  check(hv_xor_bind(ctx(), W(a), a.rows(), a.dim(), W(b), b.rows(), b.dim(), W(out)));
  return out;
}

PackedBitMatrix rotate(const PackedBitMatrix& m, std::size_t shift) {
  PackedBitMatrix out(m.rows(), m.dim());
  check(hv_rotate(ctx(), W(m), m.rows(), m.dim(), shift, W(out)));
  return out;
}

CountVector horizontal_sum(const PackedBitMatrix& m) {
  CountVector out(m.rows(), 0);
  check(hv_horizontal_sum(ctx(), W(m), m.rows(), m.dim(), out.data()));
  return out;
}

PackedBitMatrix transpose(const PackedBitMatrix& m) {
  PackedBitMatrix out(m.dim(), m.rows());
  check(hv_transpose(ctx(), W(m), m.rows(), m.dim(), W(out)));
  return out;
}

CountVector vertical_sum(const PackedBitMatrix& m) {
  CountVector out(m.dim(), 0);
  check(hv_vertical_sum(ctx(), W(m), m.rows(), m.dim(), out.data()));
  return out;
}

PackedBitMatrix majority_binarize(const CountVector& counts, std::uint64_t n, const PackedBitMatrix& tiebreak) {
  PackedBitMatrix out(1, counts.size());
  check(hv_majority_binarize(ctx(), counts.data(), counts.size(), n, W(tiebreak), tiebreak.rows(), tiebreak.dim(),
                             W(out)));
  return out;
}

// --------------------------------------------------------- encoding.hpp ----
Discretizer fit_discretizer(std::span<const double> data, std::size_t rows, std::size_t features,
                            std::size_t bins) {
  if (rows != 0 && features != 0 && bins >= 2 && data.size() != rows * features) {
    throw std::invalid_argument("fit_discretizer: data length does not match rows x features");
  }
  Discretizer d;
  d.bins = bins;
  d.min.assign(features, 0.0);
  d.max.assign(features, 0.0);
  check(hv_fit_discretizer(ctx(), data.data(), rows, features, bins, d.min.data(), d.max.data()));
  return d;
}

std::vector<std::uint32_t> discretize_matrix(std::span<const double> data, std::size_t rows, const Discretizer& d) {
  if (data.size() != rows * d.feature_count()) {
    throw std::invalid_argument("discretize_matrix: data length does not match rows x features");
  }
  std::vector<std::uint32_t> out(data.size(), 0);
  check(hv_discretize_matrix(ctx(), data.data(), rows, d.feature_count(), d.min.data(), d.max.data(), d.bins,
                             out.data()));
  return out;
}

std::vector<std::uint32_t> discretize(std::span<const double> x, const Discretizer& d) {
  if (x.size() != d.feature_count()) {
    throw std::invalid_argument("discretize: expected " + std::to_string(d.feature_count()) + " features, got " +
                                std::to_string(x.size()));
  }
  return discretize_matrix(x, 1, d);
}

static hv_binding binding_of(BindingStrategy b) {
  switch (b) {
    case BindingStrategy::kIdLevel: return HV_BIND_ID_LEVEL;
    case BindingStrategy::kPermutation: return HV_BIND_PERMUTATION;
    case BindingStrategy::kAppending: return HV_BIND_APPENDING;
  }
  throw std::logic_error("bad BindingStrategy");
}

PackedBitMatrix encode_batch(std::span<const std::uint32_t> bin_rows, std::size_t rows, const Codebook& codebook,
                             const PackedBitMatrix& tiebreak, std::size_t /*threads*/) {
  const std::size_t features = codebook.feature_count();
  if (bin_rows.size() != rows * features) {
    throw std::invalid_argument("encode_batch: bin matrix length does not match rows x features");
  }
  PackedBitMatrix out(rows, codebook.dim());
  check(hv_encode_batch(ctx(), bin_rows.data(), rows, features, W(codebook.id_vectors), W(codebook.value_vectors),
                        codebook.bin_count(), codebook.dim(), binding_of(codebook.binding), W(tiebreak),
                        tiebreak.rows(), tiebreak.dim(), W(out)));
  return out;
}

PackedBitMatrix encode(std::span<const std::uint32_t> bins, const Codebook& codebook,
                       const PackedBitMatrix& tiebreak) {
  if (bins.size() != codebook.feature_count()) {
    throw std::invalid_argument("encode: expected " + std::to_string(codebook.feature_count()) +
                                " bin indices, got " + std::to_string(bins.size()));
  }
  return encode_batch(bins, 1, codebook, tiebreak, 1);
}

// ------------------------------------------------------------ model.hpp ----
double hamming_distance_words(std::span<const std::uint32_t> a, std::span<const std::uint32_t> b, std::size_t dim) {
  double d = 0.0;
  check(hv_hamming_distance(ctx(), a.data(), b.data(), dim, &d));
  return d;
}

double hamming_distance(const PackedBitMatrix& a, std::size_t row_a, const PackedBitMatrix& b, std::size_t row_b) {
  if (a.dim() != b.dim()) {
    throw std::invalid_argument("hamming_distance: dimensions " + std::to_string(a.dim()) + " vs " +
                                std::to_string(b.dim()));
  }
  return hamming_distance_words(a.row(row_a), b.row(row_b), a.dim());
}

double cosine_similarity(std::span<const double> acc, std::span<const std::uint32_t> packed_row, std::size_t dim) {
  double s = 0.0;
  check(hv_cosine_similarity(ctx(), acc.data(), acc.size(), packed_row.data(), dim, &s));
  return s;
}

HDModel make_empty_model(const ModelConfig& config) {
  HDModel m = allocate(config);
  hv_model v = view(m);
  check(hv_make_empty_model(&v));
  return m;
}

ModelSnapshot freeze(const HDModel& model) {
  // model.cpp:246-248: the batch-start copy of the class vectors (and the
  // accumulators the cosine metric scores against)
  return ModelSnapshot{model.class_vectors, model.accumulators};
}


void HDModel::refresh_binarization(std::size_t c) {
  hv_model v = view(*this);
  check(hv_refresh_binarization(ctx(), &v, c));
}

void HDModel::refresh_binarization() {
  hv_model v = view(*this);
  check(hv_refresh_binarization(ctx(), &v, SIZE_MAX));
}

HDModel train_classical(const PackedBitMatrix& encoded, std::span<const int> labels, const ModelConfig& config) {
  ModelConfig cfg = config;
  cfg.dim = encoded.dim();
  HDModel m = allocate(cfg);
  hv_model v = view(m);
  check(hv_train_classical(ctx(), W(encoded), encoded.rows(), encoded.dim(),
                           reinterpret_cast<const int32_t*>(labels.data()), labels.size(), &v));
  return m;
}

void online_update(HDModel& model, const PackedBitMatrix& batch, std::span<const int> labels,
                   const ModelSnapshot& frozen) {
  hv_model v = view(model);
  check(hv_online_update(ctx(), &v, W(batch), batch.rows(), batch.dim(),
                         reinterpret_cast<const int32_t*>(labels.data()), labels.size(), W(frozen.class_vectors),
                         frozen.accumulators.empty() ? nullptr : frozen.accumulators.data()));
}

HDModel train_online(const PackedBitMatrix& encoded, std::span<const int> labels, std::size_t batch_size,
                     const ModelConfig& config) {
  ModelConfig cfg = config;
  cfg.dim = encoded.dim();
  HDModel m = allocate(cfg);
  hv_model v = view(m);
  check(hv_train_online(ctx(), W(encoded), encoded.rows(), encoded.dim(),
                        reinterpret_cast<const int32_t*>(labels.data()), labels.size(), batch_size, &v));
  return m;
}

std::vector<Prediction> predict(const HDModel& model, const PackedBitMatrix& encoded, std::size_t /*threads*/) {
  const std::size_t C = model.config.class_count;
  std::vector<int32_t> labels(encoded.rows());
  std::vector<double> dist(encoded.rows() * C);
  hv_model v = view(const_cast<HDModel&>(model));
  check(hv_predict(ctx(), &v, W(encoded), encoded.rows(), encoded.dim(), labels.data(), dist.data()));
  std::vector<Prediction> out(encoded.rows());
  for (std::size_t i = 0; i < out.size(); ++i) {
    out[i].label = labels[i];
    out[i].distances.assign(dist.begin() + static_cast<long>(i * C), dist.begin() + static_cast<long>((i + 1) * C));
  }
  return out;
}

// ------------------------------------------------------------- eval.hpp ----
std::vector<int> smooth_labels(std::span<const int> labels, std::size_t window) {
  std::vector<int> out(labels.size());
  check(hv_smooth_labels(ctx(), reinterpret_cast<const int32_t*>(labels.data()), labels.size(), window,
                         reinterpret_cast<int32_t*>(out.data())));
  return out;
}

EvalReport sample_metrics(std::span<const int> pred, std::span<const int> truth, int positive_class) {
  hv_eval_report r{};
  check(hv_sample_metrics(ctx(), reinterpret_cast<const int32_t*>(pred.data()), pred.size(),
                          reinterpret_cast<const int32_t*>(truth.data()), truth.size(), positive_class, &r));
  EvalReport out;
  out.tp = r.tp;
  out.fp = r.fp;
  out.tn = r.tn;
  out.fn = r.fn;
  out.accuracy = r.accuracy;
  if (r.has_tpr) out.tpr = r.tpr;
  if (r.has_ppv) out.ppv = r.ppv;
  if (r.has_f1) out.f1 = r.f1;
  return out;
}

EpisodeCounts episode_metrics(std::span<const int> pred, std::span<const int> truth, int positive_class) {
  EpisodeCounts e;
  check(hv_episode_metrics(ctx(), reinterpret_cast<const int32_t*>(pred.data()), pred.size(),
                           reinterpret_cast<const int32_t*>(truth.data()), truth.size(), positive_class, &e.detected,
                           &e.total, &e.false_positive));
  return e;
}

}  // namespace hypervec
