// golden_gen — writes golden vectors produced by the REFERENCE library.
//
// Test infrastructure only. Built by oracle/Makefile against
// oracle/_ref/libhypervec.a (compiled from /root/reference/proj/src, never
// copied) and the reference test support synth.cpp. Output: tests/golden/,
// one directory per case holding .npy arrays plus meta.txt (key=value).
// These fixtures pin both the C oracle (oracle/hv_oracle.c) and the CUDA
// engine: the reference itself cannot travel to the GPU box.
//
// Usage: golden_gen <out_dir>

#include <cstdint>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <map>
#include <sstream>
#include <span>
#include <bit>
#include <string>
#include <vector>

#include "hypervec/bitmat.hpp"
#include "hypervec/data.hpp"
#include "hypervec/encoding.hpp"
#include "hypervec/eval.hpp"
#include "hypervec/io.hpp"
#include "hypervec/kernels.hpp"
#include "hypervec/model.hpp"
#include "hypervec/rng.hpp"
#include "npy.hpp"
#include "support/synth.hpp"
#include "support/testutil.hpp"

namespace fs = std::filesystem;
using namespace hypervec;

namespace {

fs::path g_root;

struct Case {
  fs::path dir;
  std::map<std::string, std::string> meta;
  explicit Case(const std::string& name) : dir(g_root / name) { fs::create_directories(dir); }
  ~Case() {
    std::ofstream out(dir / "meta.txt");
    for (const auto& [k, v] : meta) out << k << "=" << v << "\n";
  }
  template <typename T>
  void put(const std::string& name, const std::vector<T>& v, std::vector<std::size_t> shape = {}) {
    if (shape.empty()) shape = {v.size()};
    npy::save((dir / (name + ".npy")).string(), v, shape);
  }
  void packed(const std::string& name, const PackedBitMatrix& m) {
    put(name, m.words(), {m.rows(), m.words_per_row()});
  }
  void dense(const std::string& name, const DenseBitMatrix& m) { put(name, m.bits(), {m.rows(), m.dim()}); }
  template <typename T>
  void set(const std::string& k, const T& v) { meta[k] = std::to_string(v); }
};

std::vector<std::uint64_t> to_u64(const CountVector& c) { return {c.begin(), c.end()}; }

void gen_rng() {
  Case c("rng");
  for (std::uint64_t seed : {0ull, 1ull, 42ull, 0xdeadbeefcafef00dull}) {
    Rng r(seed);
    std::vector<std::uint64_t> s(700);  // crosses two twists
    for (auto& v : s) v = r.next_u64();
    c.put("mt64_" + std::to_string(seed), s);
    Rng u(seed);
    std::vector<std::uint64_t> below(64);
    for (std::size_t i = 0; i < below.size(); ++i) below[i] = u.uniform_below(1 + i * 977);
    c.put("below_" + std::to_string(seed), below);
    Rng q(seed);
    std::vector<double> unit(64);
    for (auto& v : unit) v = q.next_unit();
    c.put("unit_" + std::to_string(seed), unit);
  }
  std::vector<std::uint64_t> sm, ds;
  for (std::uint64_t x = 0; x < 64; ++x) {
    sm.push_back(splitmix64(x * 0x9E3779B97F4A7C15ull));
    for (std::uint64_t tag = 1; tag <= 4; ++tag) ds.push_back(derive_seed(x, tag));
  }
  c.put("splitmix64", sm);
  c.put("derive_seed", ds, {64, 4});
}

void gen_codebooks() {
  Case c("codebook");
  c.packed("random_5x10240_s99", generate_random(5, 10240, 99));
  c.packed("random_3x33_s7", generate_random(3, 33, 7));
  c.packed("scale_random_16x10240_s7", generate_scale_random(16, 10240, 7));
  c.packed("scale_random_17x32_s1", generate_scale_random(17, 32, 1));
  c.packed("sandwich_8x1000_s5", generate_sandwich(8, 1000, 5));
  c.packed("sandwich_5x64_s3", generate_sandwich(5, 64, 3));
  for (auto [gname, g] : {std::pair{"random", GenerationStrategy::kRandom},
                          std::pair{"scale_random", GenerationStrategy::kScaleRandom},
                          std::pair{"sandwich", GenerationStrategy::kSandwich}}) {
    Codebook cb = make_codebook(g, BindingStrategy::kIdLevel, 12, 8, 1024, 77);
    c.packed(std::string("cb_") + gname + "_id", cb.id_vectors);
    c.packed(std::string("cb_") + gname + "_value", cb.value_vectors);
  }
}

void gen_kernels() {
  // Edge widths from testutil::edge_dims (tests/support/testutil.hpp:18-22);
  // rows capped like test_kernels.cpp rows_for().
  int idx = 0;
  for (std::size_t dim : testutil::edge_dims()) {
    Rng rng(derive_seed(1234, dim));
    const std::size_t rows = dim > 4096 ? 5 : (dim > 256 ? 19 : 37);
    Case c("kernels_" + std::to_string(idx++));
    c.set("rows", rows);
    c.set("dim", dim);
    DenseBitMatrix a = testutil::random_dense(rows, dim, rng);
    DenseBitMatrix b = testutil::random_dense(rows, dim, rng);
    DenseBitMatrix b1 = testutil::random_dense(1, dim, rng);
    PackedBitMatrix pa = pack(a), pb = pack(b), pb1 = pack(b1);
    c.dense("a", a);
    c.dense("b", b);
    c.dense("b1", b1);
    c.packed("pack_a", pa);
    c.packed("xor_ab", xor_bind(pa, pb));
    c.packed("xor_ab1", xor_bind(pa, pb1));
    std::vector<std::uint64_t> shifts = {0, 1, dim / 3, dim - 1, dim, dim + 7};
    c.put("shifts", shifts);
    for (std::size_t k = 0; k < shifts.size(); ++k) c.packed("rot_" + std::to_string(k), rotate(pa, shifts[k]));
    c.put("hsum", to_u64(horizontal_sum(pa)));
    c.packed("transpose", transpose(pa));
    c.put("vsum", to_u64(vertical_sum(pa)));
    const std::uint64_t n = 1 + rng.uniform_below(50);
    CountVector counts = testutil::random_counts(dim, n, rng);
    DenseBitMatrix tb = testutil::random_dense(1, dim, rng);
    c.set("maj_n", n);
    c.put("maj_counts", to_u64(counts));
    c.dense("maj_tiebreak", tb);
    c.packed("maj_out", majority_binarize(counts, n, pack(tb)));
  }
}

void gen_discretize() {
  Case c("discretize");
  Rng rng(41);
  const std::size_t rows = 50, features = 7;
  std::vector<double> data(rows * features);
  for (double& v : data) v = rng.next_unit() * 20.0 - 10.0;
  data[3 * features + 2] = data[0 * features + 2];  // harmless duplicates
  for (std::size_t r = 0; r < rows; ++r) data[r * features + 5] = 3.25;  // degenerate feature
  Discretizer d = fit_discretizer(data, rows, features, 16);
  c.put("data", data, {rows, features});
  c.put("min", d.min);
  c.put("max", d.max);
  c.put("bins", discretize_matrix(data, rows, d), {rows, features});
  // Out-of-range / special values against the fitted ranges.
  std::vector<double> probe = {-1e9, 1e9, 0.0, -0.0, 7.5, -7.5, 1e-300, 9.999999, -9.999999, 10.0,
                               -10.0, 3.25, 2.0, std::numeric_limits<double>::quiet_NaN()};
  std::vector<double> probe_rows;
  for (double p : probe) for (std::size_t f = 0; f < features; ++f) probe_rows.push_back(p);
  c.put("probe", probe_rows, {probe.size(), features});
  c.put("probe_bins", discretize_matrix(probe_rows, probe.size(), d), {probe.size(), features});
}

// Encode goldens: codebook regenerated from (generation, F, B, D, seed) by
// the consumer; bins + tiebreak seed + reference output stored.
void gen_encode() {
  struct Spec { const char* name; GenerationStrategy g; BindingStrategy b; std::size_t F, B, D, rows; std::uint64_t seed; };
  const Spec specs[] = {
      {"isolet", GenerationStrategy::kRandom, BindingStrategy::kIdLevel, 617, 16, 10000, 6, 101},
      {"chbmit", GenerationStrategy::kRandom, BindingStrategy::kIdLevel, 342, 16, 10000, 6, 102},
      {"mnist_1k", GenerationStrategy::kRandom, BindingStrategy::kIdLevel, 784, 16, 1024, 6, 103},
      {"uci_har", GenerationStrategy::kRandom, BindingStrategy::kIdLevel, 561, 16, 10000, 4, 104},
      {"idl_scale", GenerationStrategy::kScaleRandom, BindingStrategy::kIdLevel, 30, 16, 2048, 9, 105},
      {"idl_sandwich", GenerationStrategy::kSandwich, BindingStrategy::kIdLevel, 24, 7, 1000, 9, 106},
      {"idl_tiny", GenerationStrategy::kRandom, BindingStrategy::kIdLevel, 3, 2, 16, 8, 3},
      {"idl_f1", GenerationStrategy::kRandom, BindingStrategy::kIdLevel, 1, 4, 333, 4, 9},
      {"idl_even", GenerationStrategy::kRandom, BindingStrategy::kIdLevel, 64, 5, 33, 20, 107},
      {"perm_97", GenerationStrategy::kRandom, BindingStrategy::kPermutation, 5, 3, 97, 7, 11},
      {"perm_1000", GenerationStrategy::kScaleRandom, BindingStrategy::kPermutation, 40, 16, 1000, 6, 108},
      {"perm_10240", GenerationStrategy::kRandom, BindingStrategy::kPermutation, 100, 16, 10240, 3, 109},
      {"app_37", GenerationStrategy::kRandom, BindingStrategy::kAppending, 4, 3, 37, 6, 13},
      {"app_10000", GenerationStrategy::kRandom, BindingStrategy::kAppending, 617, 16, 10000, 3, 110},
      // more than 16 bins: the table encoder's 32-bin tables
      {"b32_chbmit", GenerationStrategy::kRandom, BindingStrategy::kIdLevel, 342, 32, 10000, 6, 111},
      {"b24_isolet", GenerationStrategy::kRandom, BindingStrategy::kIdLevel, 617, 24, 10000, 4, 112},
      {"perm_b32", GenerationStrategy::kRandom, BindingStrategy::kPermutation, 100, 32, 2048, 5, 113},
  };
  for (const Spec& s : specs) {
    Case c(std::string("encode_") + s.name);
    Codebook cb = make_codebook(s.g, s.b, s.F, s.B, s.D, s.seed);
    PackedBitMatrix tb = generate_random(1, s.D, s.seed + 1);
    Rng rng(s.seed + 2);
    std::vector<std::uint32_t> bins(s.rows * s.F);
    for (auto& v : bins) v = static_cast<std::uint32_t>(rng.uniform_below(s.B));
    c.set("generation", static_cast<int>(s.g));
    c.set("binding", static_cast<int>(s.b));
    c.set("F", s.F);
    c.set("B", s.B);
    c.set("D", s.D);
    c.set("rows", s.rows);
    c.set("seed", s.seed);
    c.set("tiebreak_seed", s.seed + 1);
    c.put("bins", bins, {s.rows, s.F});
    c.packed("out", encode_batch(bins, s.rows, cb, tb, 1));
    // checksum of the codebook words so a mismatched regeneration is obvious
    std::uint64_t h = 1469598103934665603ull;
    for (std::uint32_t w : cb.id_vectors.words()) h = (h ^ w) * 1099511628211ull;
    for (std::uint32_t w : cb.value_vectors.words()) h = (h ^ w) * 1099511628211ull;
    c.meta["codebook_fnv"] = std::to_string(h);
  }
}

// End-to-end fold on make_synth data (tests/support/synth.cpp:16-47), the
// run_fold_packed path (experiment.cpp:148-178) with explicit stages.
void gen_pipeline(const std::string& name, std::size_t rows, std::size_t features,
                  std::size_t classes, std::size_t dim, std::uint64_t seed,
                  std::vector<std::size_t> batch_sizes, double gamma) {
  Case c("pipeline_" + name);
  synth::SynthSpec spec;
  spec.rows = rows;
  spec.features = features;
  spec.classes = classes;
  spec.seed = seed;
  Dataset ds = synth::make_synth(spec);
  const std::size_t train_rows = std::min(rows - 1, std::max<std::size_t>(1, rows * 4 / 5));
  const std::size_t bins_n = 16;
  Discretizer disc = fit_discretizer(std::span<const double>(ds.X.data(), train_rows * features),
                                     train_rows, features, bins_n);
  std::vector<std::uint32_t> bins = discretize_matrix(ds.X, rows, disc);
  Codebook cb = make_codebook(GenerationStrategy::kRandom, BindingStrategy::kIdLevel, features,
                              bins_n, dim, derive_seed(seed, 1));
  PackedBitMatrix etb = generate_random(1, dim, derive_seed(seed, 2));
  PackedBitMatrix enc = encode_batch(bins, rows, cb, etb, 4);
  c.set("rows", rows);
  c.set("features", features);
  c.set("classes", classes);
  c.set("dim", dim);
  c.set("seed", seed);
  c.set("train_rows", train_rows);
  c.set("gamma_bits", std::bit_cast<std::uint64_t>(gamma));
  c.put("X", ds.X, {rows, features});
  c.put("y", ds.y);
  c.put("min", disc.min);
  c.put("max", disc.max);
  c.put("bins", bins, {rows, features});
  c.packed("encoded", enc);

  PackedBitMatrix train(train_rows, dim), test(rows - train_rows, dim);
  for (std::size_t r = 0; r < rows; ++r) {
    auto src = enc.row(r);
    auto dst = r < train_rows ? train.row(r) : test.row(r - train_rows);
    std::copy(src.begin(), src.end(), dst.begin());
  }
  std::vector<int> ytrain(ds.y.begin(), ds.y.begin() + static_cast<long>(train_rows));
  ModelConfig cfg{classes, dim, Metric::kHamming, gamma, seed};
  HDModel cl = train_classical(train, ytrain, cfg);
  c.put("classical_acc", cl.accumulators, {classes, dim});
  c.put("classical_weight", cl.class_weight);
  c.put("classical_counts", cl.sample_counts);
  c.packed("classical_cv", cl.class_vectors);
  c.packed("model_tiebreak", cl.tiebreak);
  auto preds = predict(cl, test, 3);
  std::vector<int> pl;
  std::vector<double> pd;
  for (const auto& p : preds) {
    pl.push_back(p.label);
    pd.insert(pd.end(), p.distances.begin(), p.distances.end());
  }
  c.put("classical_pred", pl);
  c.put("classical_dist", pd, {preds.size(), classes});
  std::vector<std::uint64_t> bs(batch_sizes.begin(), batch_sizes.end());
  c.put("batch_sizes", bs);
  for (std::size_t b : batch_sizes) {
    HDModel on = train_online(train, ytrain, b, cfg);
    const std::string k = "online_b" + std::to_string(b);
    c.put(k + "_acc", on.accumulators, {classes, dim});
    c.put(k + "_weight", on.class_weight);
    c.put(k + "_counts", on.sample_counts);
    c.packed(k + "_cv", on.class_vectors);
    auto op = predict(on, test, 2);
    std::vector<int> ol;
    for (const auto& p : op) ol.push_back(p.label);
    c.put(k + "_pred", ol);
  }
  // cosine metric on the classical model (f2 row): labels + scores
  ModelConfig ccfg = cfg;
  ccfg.metric = Metric::kCosine;
  HDModel cc = train_classical(train, ytrain, ccfg);
  auto cp = predict(cc, test, 1);
  std::vector<int> cl2;
  std::vector<double> cd;
  for (const auto& p : cp) {
    cl2.push_back(p.label);
    cd.insert(cd.end(), p.distances.begin(), p.distances.end());
  }
  c.put("cosine_pred", cl2);
  c.put("cosine_dist", cd, {cp.size(), classes});
  HDModel con = train_online(train, ytrain, batch_sizes.front(), ccfg);
  c.put("cosine_online_acc", con.accumulators, {classes, dim});
  c.put("cosine_online_weight", con.class_weight);
  c.packed("cosine_online_cv", con.class_vectors);
}

// FNV-1a 64 over 32-bit words / 64-bit patterns: row and class digests for
// the large pipelines, whose full arrays would be too big to commit.
std::uint64_t fnv_words(std::span<const std::uint32_t> w) {
  std::uint64_t h = 1469598103934665603ull;
  for (std::uint32_t x : w) h = (h ^ x) * 1099511628211ull;
  return h;
}
std::uint64_t fnv_doubles(std::span<const double> v) {
  std::uint64_t h = 1469598103934665603ull;
  for (double d : v) h = (h ^ std::bit_cast<std::uint64_t>(d)) * 1099511628211ull;
  return h;
}

// run_fold_packed at D = 10000 and the benchmark shapes (UCI-HAR, ISOLET,
// MNIST at D = 20000), thousands of rows: inputs are regenerated by the
// oracle's make_synth restatement (pinned by the small pipelines' X), so only
// digests of X / bins / encoded rows / accumulators are stored, plus the
// small outputs (class vectors, weights, counts, labels, distances) in full.
void gen_pipeline_big(const std::string& name, std::size_t rows, std::size_t features, std::size_t classes,
                      std::size_t dim, std::uint64_t seed, std::vector<std::size_t> batch_sizes, double gamma,
                      std::size_t threads) {
  Case c("bigpipe_" + name);
  synth::SynthSpec spec;
  spec.rows = rows;
  spec.features = features;
  spec.classes = classes;
  spec.seed = seed;
  Dataset ds = synth::make_synth(spec);
  const std::size_t train_rows = std::min(rows - 1, std::max<std::size_t>(1, rows * 4 / 5));
  const std::size_t bins_n = 16;
  Discretizer disc = fit_discretizer(std::span<const double>(ds.X.data(), train_rows * features), train_rows,
                                     features, bins_n);
  std::vector<std::uint32_t> bins = discretize_matrix(ds.X, rows, disc);
  Codebook cb = make_codebook(GenerationStrategy::kRandom, BindingStrategy::kIdLevel, features, bins_n, dim,
                              derive_seed(seed, 1));
  PackedBitMatrix etb = generate_random(1, dim, derive_seed(seed, 2));
  PackedBitMatrix enc = encode_batch(bins, rows, cb, etb, threads);
  c.set("rows", rows);
  c.set("features", features);
  c.set("classes", classes);
  c.set("dim", dim);
  c.set("seed", seed);
  c.set("train_rows", train_rows);
  c.set("gamma_bits", std::bit_cast<std::uint64_t>(gamma));
  std::vector<std::uint64_t> xh(rows), bh(rows), eh(rows);
  for (std::size_t r = 0; r < rows; ++r) {
    xh[r] = fnv_doubles(std::span<const double>(ds.X.data() + r * features, features));
    bh[r] = fnv_words(std::span<const std::uint32_t>(bins.data() + r * features, features));
    eh[r] = fnv_words(enc.row(r));
  }
  c.put("X_fnv", xh);
  c.put("bins_fnv", bh);
  c.put("encoded_fnv", eh);
  c.put("y", ds.y);
  c.put("min", disc.min);
  c.put("max", disc.max);

  PackedBitMatrix train(train_rows, dim), test(rows - train_rows, dim);
  for (std::size_t r = 0; r < rows; ++r) {
    auto src = enc.row(r);
    auto dst = r < train_rows ? train.row(r) : test.row(r - train_rows);
    std::copy(src.begin(), src.end(), dst.begin());
  }
  std::vector<int> ytrain(ds.y.begin(), ds.y.begin() + static_cast<long>(train_rows));
  ModelConfig cfg{classes, dim, Metric::kHamming, gamma, seed};
  auto acc_fnv = [&](const HDModel& m) {
    std::vector<std::uint64_t> h(classes);
    for (std::size_t k = 0; k < classes; ++k) {
      h[k] = fnv_doubles(std::span<const double>(m.accumulators.data() + k * dim, dim));
    }
    return h;
  };
  HDModel cl = train_classical(train, ytrain, cfg);
  c.put("classical_acc_fnv", acc_fnv(cl));
  c.put("classical_weight", cl.class_weight);
  c.put("classical_counts", cl.sample_counts);
  c.packed("classical_cv", cl.class_vectors);
  c.packed("model_tiebreak", cl.tiebreak);
  auto preds = predict(cl, test, threads);
  std::vector<int> pl;
  std::vector<double> pd;
  for (const auto& p : preds) {
    pl.push_back(p.label);
    pd.insert(pd.end(), p.distances.begin(), p.distances.end());
  }
  c.put("classical_pred", pl);
  c.put("classical_dist", pd, {preds.size(), classes});
  std::vector<std::uint64_t> bs(batch_sizes.begin(), batch_sizes.end());
  c.put("batch_sizes", bs);
  for (std::size_t b : batch_sizes) {
    HDModel on = train_online(train, ytrain, b, cfg);
    const std::string k = "online_b" + std::to_string(b);
    c.put(k + "_acc_fnv", acc_fnv(on));
    c.put(k + "_weight", on.class_weight);
    c.put(k + "_counts", on.sample_counts);
    c.packed(k + "_cv", on.class_vectors);
    auto op = predict(on, test, threads);
    std::vector<int> ol;
    for (const auto& p : op) ol.push_back(p.label);
    c.put(k + "_pred", ol);
  }
}

// One online_update on random packed state (test_model.cpp:180-205 shape).
void gen_online_update() {
  Case c("online_update");
  Rng rng(53);
  const std::size_t dim = 300, classes = 4;
  DenseBitMatrix base = testutil::random_dense(20, dim, rng);
  std::vector<int> base_y(20);
  for (int& v : base_y) v = static_cast<int>(rng.uniform_below(classes));
  ModelConfig cfg{classes, dim, Metric::kHamming, 0.25 + rng.next_unit(), rng.next_u64()};
  HDModel m = train_classical(pack(base), base_y, cfg);
  c.dense("base", base);
  c.put("base_y", base_y);
  c.set("gamma_bits", std::bit_cast<std::uint64_t>(cfg.gamma));
  c.set("seed", cfg.seed);
  c.set("classes", classes);
  c.set("dim", dim);
  DenseBitMatrix batch = testutil::random_dense(16, dim, rng);
  std::vector<int> y(16);
  for (int& v : y) v = static_cast<int>(rng.uniform_below(classes));
  online_update(m, pack(batch), y, freeze(m));
  c.dense("batch", batch);
  c.put("y", y);
  c.put("acc", m.accumulators, {classes, dim});
  c.put("weight", m.class_weight);
  c.put("counts", m.sample_counts);
  c.packed("cv", m.class_vectors);
}

void gen_synth() {
  Case c("synth");
  synth::SynthSpec spec;
  spec.rows = 64;
  spec.features = 30;
  spec.classes = 5;
  spec.seed = 501;
  Dataset ds = synth::make_synth(spec);
  c.put("X", ds.X, {ds.rows, ds.features});
  c.put("y", ds.y);
}

// eval.cpp:12-116 on sequences shaped like concatenated fold predictions:
// seizure-like runs, glitches, multi-class labels, edge lengths and windows.
void gen_eval() {
  Rng rng(777);
  const std::vector<std::size_t> lengths = {0, 1, 2, 3, 7, 64, 1000, 4099};
  const std::vector<std::size_t> windows = {1, 3, 5, 9, 31, 101};
  int k = 0;
  for (std::size_t n : lengths) {
    for (int variant = 0; variant < 3; ++variant) {
      Case c("eval_" + std::to_string(k++));
      std::vector<int> truth(n), pred(n);
      // truth: runs of positives (variant 0/1) or 5-class labels (variant 2)
      int cur = 0;
      for (std::size_t i = 0; i < n; ++i) {
        if (variant == 2) {
          truth[i] = static_cast<int>(rng.uniform_below(5));
        } else {
          if (rng.uniform_below(variant == 0 ? 40 : 6) == 0) cur ^= 1;
          truth[i] = cur;
        }
        const bool flip = rng.uniform_below(variant == 1 ? 3 : 10) == 0;
        pred[i] = variant == 2 ? (flip ? static_cast<int>(rng.uniform_below(5)) : truth[i])
                               : (flip ? 1 - truth[i] : truth[i]);
      }
      c.put("pred", pred);
      c.put("truth", truth);
      const int positive = variant == 2 ? 2 : 1;
      c.set("positive", positive);
      std::vector<double> ratios = {std::numeric_limits<double>::quiet_NaN(), std::numeric_limits<double>::quiet_NaN(),
                                    std::numeric_limits<double>::quiet_NaN(), std::numeric_limits<double>::quiet_NaN()};
      if (n > 0) {
        const EvalReport r = sample_metrics(pred, truth, positive);
        c.put("counts", std::vector<std::uint64_t>{r.tp, r.fp, r.tn, r.fn});
        ratios[0] = r.accuracy;
        if (r.tpr) ratios[1] = *r.tpr;
        if (r.ppv) ratios[2] = *r.ppv;
        if (r.f1) ratios[3] = *r.f1;
        c.put("ratios", ratios);
      }
      const EpisodeCounts e = episode_metrics(pred, truth, positive);
      c.put("episodes", std::vector<std::uint64_t>{e.detected, e.total, e.false_positive});
      if (variant != 2) {
        for (std::size_t w : windows) c.put("smooth_" + std::to_string(w), smooth_labels(pred, w));
      }
    }
  }
}

std::vector<std::uint8_t> bytes_of(const std::string& s) { return {s.begin(), s.end()}; }

// io.cpp:85-107 (HVPB), encoding.cpp:313-330 (HVCB), model.cpp:322-337 (HVMD)
// written by the reference for the "odd" pipeline (pipeline_odd inputs) and
// for models whose gamma exercises the JSON number formatting.
void gen_containers() {
  Case c("containers");
  synth::SynthSpec spec;
  spec.rows = 157;
  spec.features = 13;
  spec.classes = 3;
  spec.seed = 12;
  Dataset ds = synth::make_synth(spec);
  const std::size_t rows = 157, F = 13, C = 3, D = 1000, train_rows = 125;
  Discretizer disc = fit_discretizer(std::span<const double>(ds.X.data(), train_rows * F), train_rows, F, 16);
  std::vector<std::uint32_t> bins = discretize_matrix(ds.X, rows, disc);
  Codebook cb = make_codebook(GenerationStrategy::kRandom, BindingStrategy::kIdLevel, F, 16, D, derive_seed(12, 1));
  PackedBitMatrix etb = generate_random(1, D, derive_seed(12, 2));
  PackedBitMatrix enc = encode_batch(bins, rows, cb, etb, 2);
  PackedBitMatrix train(train_rows, D);
  for (std::size_t r = 0; r < train_rows; ++r) {
    auto src = enc.row(r);
    std::copy(src.begin(), src.end(), train.row(r).begin());
  }
  std::vector<int> ytrain(ds.y.begin(), ds.y.begin() + static_cast<long>(train_rows));
  auto dump = [&](const std::string& key, auto&& writer) {
    std::ostringstream out(std::ios::binary);
    writer(out);
    c.put(key, bytes_of(out.str()));
  };
  dump("hvpb_encoded", [&](std::ostream& o) { io::write_packed(o, enc); });
  dump("hvpb_empty", [&](std::ostream& o) { io::write_packed(o, PackedBitMatrix(0, 37)); });
  dump("hvcb_random", [&](std::ostream& o) { save_codebook(cb, o); });
  Codebook cb2 = make_codebook(GenerationStrategy::kSandwich, BindingStrategy::kPermutation, 5, 4, 64, 99);
  dump("hvcb_sandwich_perm", [&](std::ostream& o) { save_codebook(cb2, o); });
  ModelConfig cfg{C, D, Metric::kHamming, 0.6, 12};
  dump("hvmd_classical", [&](std::ostream& o) { save_model(train_classical(train, ytrain, cfg), o); });
  dump("hvmd_online_b5", [&](std::ostream& o) { save_model(train_online(train, ytrain, 5, cfg), o); });
  const std::vector<double> gammas = {1.0, 0.1, 1e-05, 123.456, 2.5e-300, 0.30000000000000004, 1e16, 7.0,
                                      1e15, 1e-4, 123456789012345.6, 0.5, 1e300, 5e-324, 0.0};
  c.put("gammas", gammas);
  for (std::size_t g = 0; g < gammas.size(); ++g) {
    ModelConfig gc{2, 40, g % 2 ? Metric::kCosine : Metric::kHamming, gammas[g], 1000 + g};
    dump("hvmd_gamma_" + std::to_string(g), [&](std::ostream& o) { save_model(make_empty_model(gc), o); });
  }
}

}  // namespace

int main(int argc, char** argv) {
  if (argc != 2) {
    std::cerr << "usage: golden_gen <out_dir>\n";
    return 2;
  }
  g_root = argv[1];
  fs::create_directories(g_root);
  gen_rng();
  gen_codebooks();
  gen_kernels();
  gen_discretize();
  gen_encode();
  gen_pipeline("small", 300, 30, 5, 2048, 11, {1, 7, 64, 1024}, 1.0);
  gen_pipeline("odd", 157, 13, 3, 1000, 12, {5, 50}, 0.6);
  gen_pipeline("isolet", 160, 617, 26, 2000, 13, {32}, 1.0);
  gen_pipeline_big("har_d10k", 12000, 561, 6, 10000, 21, {256, 1024, 8192}, 1.0, 8);
  gen_pipeline_big("isolet_d10k", 2500, 617, 26, 10000, 22, {1024}, 1.0, 8);
  gen_pipeline_big("mnist_d20k", 3000, 784, 10, 20000, 23, {1024}, 0.8, 8);
  gen_pipeline_big("mnist_d1k", 6000, 784, 10, 1024, 24, {1024, 8192}, 1.0, 8);
  gen_online_update();
  gen_synth();
  gen_eval();
  gen_containers();
  std::cout << "golden vectors written to " << g_root << "\n";
  return 0;
}
