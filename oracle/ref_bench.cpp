// ref_bench — times the UNMODIFIED reference library on the bench workload.
//
// Test/bench infrastructure only: this is the CPU baseline of bench.py
// (cpu_baseline leg and `bench.py --impl reference`). It links
// oracle/_ref/libhypervec.a, compiled from /root/reference/proj/src with the
// reference's own Release flags (-O3 -DNDEBUG -mpopcnt, CMakeLists.txt:6-19),
// and calls the reference's public API exactly as run_bench does
// (experiment.cpp:439-501): encode_batch(threads) -> train_classical |
// train_online -> predict(threads).
//
// The workload is the shared counter-based generator (include/hvb200_synth.h)
// on rows [0, rows) of the configured dataset: the first 80 % train, the rest
// test (single_split, data.cpp:245-257).
//
// Prints one JSON object on stdout.

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "hvb200_synth.h"
#include "hypervec/encoding.hpp"
#include "hypervec/model.hpp"
#include "hypervec/rng.hpp"

using namespace hypervec;

namespace {

double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

struct Args {
  std::size_t features = 342, classes = 2, dim = 10000, rows = 4096, bins = 16, threads = 0;
  std::size_t batch = 1024, reps = 1;
  int label_kind = HVS_LABELS_CHBMIT;
  std::string trainer = "classical";
  std::uint64_t seed = 1, data_seed = 7;
};

Args parse(int argc, char** argv) {
  Args a;
  for (int i = 1; i + 1 < argc; i += 2) {
    const std::string k = argv[i];
    const char* v = argv[i + 1];
    if (k == "--features") a.features = std::strtoull(v, nullptr, 10);
    else if (k == "--classes") a.classes = std::strtoull(v, nullptr, 10);
    else if (k == "--dim") a.dim = std::strtoull(v, nullptr, 10);
    else if (k == "--rows") a.rows = std::strtoull(v, nullptr, 10);
    else if (k == "--bins") a.bins = std::strtoull(v, nullptr, 10);
    else if (k == "--threads") a.threads = std::strtoull(v, nullptr, 10);
    else if (k == "--batch") a.batch = std::strtoull(v, nullptr, 10);
    else if (k == "--reps") a.reps = std::strtoull(v, nullptr, 10);
    else if (k == "--labels") a.label_kind = std::string(v) == "chbmit" ? HVS_LABELS_CHBMIT : HVS_LABELS_MOD;
    else if (k == "--trainer") a.trainer = v;
    else if (k == "--seed") a.seed = std::strtoull(v, nullptr, 10);
    else if (k == "--data-seed") a.data_seed = std::strtoull(v, nullptr, 10);
    else {
      std::fprintf(stderr, "unknown flag %s\n", k.c_str());
      std::exit(2);
    }
  }
  if (a.threads == 0) a.threads = std::max(1u, std::thread::hardware_concurrency());
  return a;
}

}  // namespace

int main(int argc, char** argv) {
  const Args a = parse(argc, argv);
  const std::size_t n = a.rows;
  const std::size_t train_rows = std::min(n - 1, std::max<std::size_t>(1, n * 4 / 5));
  const std::size_t test_rows = n - train_rows;

  std::vector<int> y(n);
  std::vector<std::uint32_t> bins(n * a.features);
  for (std::size_t i = 0; i < n; ++i) {
    y[i] = hvs_label(i, static_cast<std::uint32_t>(a.classes), a.label_kind);
    for (std::size_t f = 0; f < a.features; ++f) {
      bins[i * a.features + f] = hvs_bin(i, static_cast<std::uint32_t>(f),
                                         static_cast<std::uint32_t>(a.features), y[i],
                                         static_cast<std::uint32_t>(a.bins), a.data_seed);
    }
  }
  // Seed substreams as build_context (experiment.cpp:119-144).
  const Codebook cb = make_codebook(GenerationStrategy::kRandom, BindingStrategy::kIdLevel,
                                    a.features, a.bins, a.dim, derive_seed(a.seed, 1));
  const PackedBitMatrix etb = generate_random(1, a.dim, derive_seed(a.seed, 2));
  const ModelConfig cfg{a.classes, a.dim, Metric::kHamming, 1.0, a.seed};
  std::span<const std::uint32_t> all(bins);
  std::vector<int> ytrain(y.begin(), y.begin() + static_cast<long>(train_rows));

  double t_enc = 0, t_train = 0, t_pred = 0;
  long checksum = 0;
  for (std::size_t rep = 0; rep < a.reps; ++rep) {
    double t0 = now();
    PackedBitMatrix enc_train = encode_batch(all.subspan(0, train_rows * a.features), train_rows, cb, etb, a.threads);
    PackedBitMatrix enc_test = encode_batch(all.subspan(train_rows * a.features), test_rows, cb, etb, a.threads);
    double t1 = now();
    HDModel model = a.trainer == "online" ? train_online(enc_train, ytrain, a.batch, cfg)
                                          : train_classical(enc_train, ytrain, cfg);
    double t2 = now();
    std::vector<Prediction> preds = predict(model, enc_test, a.threads);
    double t3 = now();
    t_enc += t1 - t0;
    t_train += t2 - t1;
    t_pred += t3 - t2;
    for (std::size_t i = 0; i < preds.size(); ++i) checksum += preds[i].label * static_cast<long>(i + 1);
  }
  const double total = t_enc + t_train + t_pred;
  std::printf(
      "{\"rows\": %zu, \"train_rows\": %zu, \"test_rows\": %zu, \"features\": %zu, \"classes\": %zu, "
      "\"dim\": %zu, \"threads\": %zu, \"trainer\": \"%s\", \"reps\": %zu, \"encode_s\": %.6f, "
      "\"train_s\": %.6f, \"predict_s\": %.6f, \"total_s\": %.6f, \"dp_per_s\": %.3f, \"label_checksum\": %ld}\n",
      n, train_rows, test_rows, a.features, a.classes, a.dim, a.threads, a.trainer.c_str(), a.reps,
      t_enc, t_train, t_pred, total, static_cast<double>(n * a.reps) / total, checksum);
  return 0;
}
