/*
 * hvb200.h — C ABI of the B200 hypervector engine (libhvb200.so).
 *
 * Drop-in boundary for the hot path of the reference C++ library
 * "hypervec" (/root/reference/proj). The reference has no FFI of its own: its
 * boundary is the C++ header API in include/hypervec/{kernels,encoding,model}.hpp.
 * Every host entry point below replaces exactly one reference function and is
 * documented with the reference declaration it stands in for (file:line). A
 * C++ shim (dropin/hypervec_gpu.cpp) re-exposes the original hypervec::
 * signatures on top of these symbols; INTEGRATION.md shows the ctypes/C++
 * bindings.
 *
 * Conventions
 *  - Plain pointers and sizes; no C++ or torch types.
 *  - Packed hypervector matrices use the reference layout verbatim
 *    (bitmat.hpp:15-32): `rows` x ceil(dim/32) little-endian uint32 words,
 *    row-major, bit j of a row at word j/32 position j%32, padding bits zero.
 *  - Dense bit matrices: one byte (0/1) per bit, rows x dim row-major.
 *  - Labels are int32 (the reference's `int`).
 *  - `hv_*` entry points take HOST pointers (caller-owned), copy to the
 *    device, run the sm_100a kernels on the context's stream and copy back
 *    before returning (synchronous).
 *  - `hv_dev_*` entry points take DEVICE pointers and only enqueue work on
 *    the context's stream (asynchronous); data-dependent errors (bad bin,
 *    bad label, non-binary byte) are latched in the context and reported by
 *    hv_dev_check().
 *  - Every call returns an hv_status; the message of the last failure on the
 *    calling thread is available from hv_last_error(). Status codes map onto
 *    the reference's exception types:
 *      HV_ERR_INVALID_ARGUMENT -> std::invalid_argument
 *      HV_ERR_DOMAIN           -> std::domain_error
 *      HV_ERR_LOGIC            -> std::logic_error
 *      HV_ERR_CUDA / HV_ERR_NO_DEVICE -> std::runtime_error
 *    and invalid_argument messages reproduce the reference's wording.
 *  - There is no CPU fallback: without a usable sm_100 device every compute
 *    entry point fails with HV_ERR_NO_DEVICE.
 */
#ifndef HVB200_H
#define HVB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HVB200_ABI_VERSION 1

typedef enum hv_status {
  HV_OK = 0,
  HV_ERR_INVALID_ARGUMENT = 1,
  HV_ERR_DOMAIN = 2,
  HV_ERR_LOGIC = 3,
  HV_ERR_CUDA = 4,
  HV_ERR_NO_DEVICE = 5,
  HV_ERR_RUNTIME = 6
} hv_status;

/* encoding.hpp:17-18 */
typedef enum hv_generation { HV_GEN_RANDOM = 0, HV_GEN_SCALE_RANDOM = 1, HV_GEN_SANDWICH = 2 } hv_generation;
typedef enum hv_binding { HV_BIND_ID_LEVEL = 0, HV_BIND_PERMUTATION = 1, HV_BIND_APPENDING = 2 } hv_binding;
/* model.hpp:17 */
typedef enum hv_metric { HV_METRIC_HAMMING = 0, HV_METRIC_COSINE = 1 } hv_metric;

typedef struct hv_context hv_context;

/* ---- library / context ------------------------------------------------ */
int hv_abi_version(void);
const char* hv_last_error(void);
/* bitmat.hpp:30-32 PackedBitMatrix::words_per_row_for */
size_t hv_words_per_row(size_t dim);
/* Number of kernels this library has launched in this process (bench evidence). */
uint64_t hv_kernel_launch_count(void);

hv_status hv_context_create(int device, hv_context** out);
void hv_context_destroy(hv_context* ctx);
/* Route hv_dev_* work onto an existing cudaStream_t (NULL = the context's own stream;
 * pass cudaStreamLegacy, (void*)0x1, for the legacy default stream). */
hv_status hv_context_set_stream(hv_context* ctx, void* cuda_stream);
void* hv_context_stream(hv_context* ctx);
hv_status hv_context_synchronize(hv_context* ctx);

/* ---- RNG and codebooks: host code, bit-identical to the reference ------ */
/* rng.hpp:14-24 */
uint64_t hv_splitmix64(uint64_t x);
uint64_t hv_derive_seed(uint64_t seed, uint64_t tag);
/* encoding.hpp:49-60 (generate_random / generate_scale_random / generate_sandwich);
 * out: count x ceil(dim/32) words */
hv_status hv_generate_random(size_t count, size_t dim, uint64_t seed, uint32_t* out);
hv_status hv_generate_scale_random(size_t bins, size_t dim, uint64_t seed, uint32_t* out);
hv_status hv_generate_sandwich(size_t bins, size_t dim, uint64_t seed, uint32_t* out);
/* encoding.hpp:77-79 make_codebook: id_out F x W, value_out B x W */
hv_status hv_make_codebook(hv_generation generation, size_t features, size_t bins, size_t dim,
                           uint64_t seed, uint32_t* id_out, uint32_t* value_out);

/* ---- kernels.hpp (host pointers) --------------------------------------- */
/* kernels.hpp:16-18 pack */
hv_status hv_pack(hv_context* ctx, const uint8_t* dense, size_t rows, size_t dim, uint32_t* out);
/* kernels.hpp:20-21 unpack */
hv_status hv_unpack(hv_context* ctx, const uint32_t* words, size_t rows, size_t dim, uint8_t* out);
/* kernels.hpp:23-25 xor_bind (b_rows == a_rows or 1 = broadcast) */
hv_status hv_xor_bind(hv_context* ctx, const uint32_t* a, size_t a_rows, size_t a_dim,
                      const uint32_t* b, size_t b_rows, size_t b_dim, uint32_t* out);
/* kernels.hpp:27-29 rotate */
hv_status hv_rotate(hv_context* ctx, const uint32_t* m, size_t rows, size_t dim, size_t shift,
                    uint32_t* out);
/* kernels.hpp:31-32 horizontal_sum */
hv_status hv_horizontal_sum(hv_context* ctx, const uint32_t* m, size_t rows, size_t dim,
                            uint64_t* out);
/* kernels.hpp:34-36 transpose: out is dim x ceil(rows/32) words */
hv_status hv_transpose(hv_context* ctx, const uint32_t* m, size_t rows, size_t dim, uint32_t* out);
/* kernels.hpp:38-40 vertical_sum: out has dim counts */
hv_status hv_vertical_sum(hv_context* ctx, const uint32_t* m, size_t rows, size_t dim,
                          uint64_t* out);
/* kernels.hpp:42-46 majority_binarize: tiebreak must be 1 x dim */
hv_status hv_majority_binarize(hv_context* ctx, const uint64_t* counts, size_t dim, uint64_t n,
                               const uint32_t* tiebreak, size_t tiebreak_rows,
                               size_t tiebreak_dim, uint32_t* out);

/* ---- encoding.hpp (host pointers) -------------------------------------- */
/* encoding.hpp:37-40 fit_discretizer */
hv_status hv_fit_discretizer(hv_context* ctx, const double* data, size_t rows, size_t features,
                             size_t bins, double* min_out, double* max_out);
/* encoding.hpp:45-47 discretize_matrix (discretize = one row) */
hv_status hv_discretize_matrix(hv_context* ctx, const double* data, size_t rows, size_t features,
                               const double* min, const double* max, size_t bins, uint32_t* out);
/* encoding.hpp:81-93 encode / encode_batch. id_vectors F x W, value_vectors B x W,
 * tiebreak tiebreak_rows x ceil(tiebreak_dim/32) (must be 1 x dim). */
hv_status hv_encode_batch(hv_context* ctx, const uint32_t* bin_rows, size_t rows, size_t features,
                          const uint32_t* id_vectors, const uint32_t* value_vectors, size_t bins,
                          size_t dim, hv_binding binding, const uint32_t* tiebreak,
                          size_t tiebreak_rows, size_t tiebreak_dim, uint32_t* out);

/* ---- model.hpp (host pointers) ----------------------------------------- */
/* model.hpp:22-56 ModelConfig + HDModel state; arrays are caller-owned host
 * memory of the sizes noted. */
typedef struct hv_model {
  size_t class_count;
  size_t dim;
  hv_metric metric;
  double gamma;
  uint64_t seed;
  double* accumulators;    /* class_count x dim */
  double* class_weight;    /* class_count */
  uint64_t* sample_counts; /* class_count */
  uint32_t* class_vectors; /* class_count x ceil(dim/32) */
  uint32_t* tiebreak;      /* 1 x ceil(dim/32) */
} hv_model;

/* model.cpp:198-217 make_empty_model (validates config, fills the arrays) */
hv_status hv_make_empty_model(hv_model* model);
/* model.hpp:53-55 HDModel::refresh_binarization (class_index = SIZE_MAX: all) */
hv_status hv_refresh_binarization(hv_context* ctx, hv_model* model, size_t class_index);
/* model.hpp:81-82 train_classical (model->dim is set from dim) */
hv_status hv_train_classical(hv_context* ctx, const uint32_t* encoded, size_t rows, size_t dim,
                             const int32_t* labels, size_t n_labels, hv_model* model);
/* model.hpp:97-98 online_update against a frozen snapshot (model.hpp:86-91):
 * snapshot_class_vectors class_count x W, snapshot_accumulators (cosine only, nullable). */
hv_status hv_online_update(hv_context* ctx, hv_model* model, const uint32_t* batch, size_t rows,
                           size_t dim, const int32_t* labels, size_t n_labels,
                           const uint32_t* snapshot_class_vectors,
                           const double* snapshot_accumulators);
/* model.hpp:104-105 train_online */
hv_status hv_train_online(hv_context* ctx, const uint32_t* encoded, size_t rows, size_t dim,
                          const int32_t* labels, size_t n_labels, size_t batch_size,
                          hv_model* model);
/* model.hpp:110-111 predict: labels_out rows; distances_out rows x class_count (nullable) */
hv_status hv_predict(hv_context* ctx, const hv_model* model, const uint32_t* encoded,
                     size_t rows, size_t dim, int32_t* labels_out, double* distances_out);
/* ---- one fold of the reference pipeline (experiment.cpp:159-177) ------- */
/* run_fold_packed minus discretize: encode_batch(train) + encode_batch(test)
 * -> train_classical -> predict, with the encoded hypervectors kept in HBM
 * (they never cross PCIe). Split in two calls so a data-parallel caller can
 * all-reduce the class counts in between (hv_fold_counts). */
typedef struct hv_fold hv_fold;
hv_status hv_fold_encode_train(hv_context* ctx, const uint32_t* train_bins, size_t train_rows,
                               const int32_t* train_labels, const uint32_t* test_bins,
                               size_t test_rows, size_t features, const uint32_t* id_vectors,
                               const uint32_t* value_vectors, size_t bins, size_t dim,
                               const uint32_t* encode_tiebreak, size_t class_count, hv_fold** out);
/* device pointers of the fold's class counts (class_count x 32*W uint32) and class rows (uint64) */
hv_status hv_fold_counts(hv_fold* fold, void** counts_dev, void** class_rows_dev);
/* binarise with the model tiebreak (1 x W host words) and predict the test rows into labels_out (host) */
hv_status hv_fold_predict(hv_context* ctx, hv_fold* fold, const uint32_t* model_tiebreak, int32_t* labels_out);
void hv_fold_destroy(hv_fold* fold);

/* ---- HBM-resident datasets: whole folds from fp64 features ---------------
 * run_fold_packed (experiment.cpp:148-178) with the feature matrix resident
 * across folds (time-series / leave-one-out splits re-fit and re-encode per
 * fold without re-uploading): fit_discretizer on the train rows, discretize
 * train and test rows, encode, train (classical, or online with batch_size),
 * predict the test rows. train_idx / test_idx are host arrays of row indices
 * (any order / subset); labels_out gets n_test labels; min_out / max_out
 * (nullable, features doubles) the fitted discretizer. */
typedef struct hv_dataset hv_dataset;
hv_status hv_dataset_create(hv_context* ctx, const double* X, size_t rows, size_t features,
                            const int32_t* labels, hv_dataset** out);
void hv_dataset_destroy(hv_dataset* ds);
hv_status hv_dataset_fold(hv_context* ctx, const hv_dataset* ds, const uint64_t* train_idx,
                          size_t n_train, const uint64_t* test_idx, size_t n_test, size_t bins,
                          const uint32_t* id_vectors, const uint32_t* value_vectors, size_t dim,
                          hv_binding binding, const uint32_t* encode_tiebreak, size_t class_count,
                          hv_metric metric, double gamma, const uint32_t* model_tiebreak, int online,
                          size_t batch_size, int32_t* labels_out, double* min_out, double* max_out);

/* ---- evaluation of concatenated predictions (eval.hpp:16-74) -------------
 * EvalReport (eval.hpp:26-37): confusion counts against one positive class,
 * accuracy over exact matches, and ratios that are ABSENT (has_* = 0, value
 * NaN) when their denominator is zero, plus episode counts (eval.hpp:13-17). */
typedef struct hv_eval_report {
  uint64_t tp, fp, tn, fn;
  double accuracy, tpr, ppv, f1;
  int has_tpr, has_ppv, has_f1;
  uint64_t episodes_detected, episodes_total, episodes_false_positive;
} hv_eval_report;
/* eval.hpp:44 smooth_labels (eval.cpp:12-37): centred majority over `window`
 * in-bounds samples, ties -> 1; INVALID_ARGUMENT for an even/zero window or a
 * non-binary label (first index, reference messages). Host arrays. */
hv_status hv_smooth_labels(hv_context* ctx, const int32_t* labels, size_t n, size_t window, int32_t* out);
/* eval.hpp:48 sample_metrics (eval.cpp:39-77); episode fields left zero. */
hv_status hv_sample_metrics(hv_context* ctx, const int32_t* pred, size_t n_pred, const int32_t* truth,
                            size_t n_truth, int positive_class, hv_eval_report* report);
/* eval.hpp:52 episode_metrics (eval.cpp:79-116). */
hv_status hv_episode_metrics(hv_context* ctx, const int32_t* pred, size_t n_pred, const int32_t* truth,
                             size_t n_truth, int positive_class, uint64_t* detected, uint64_t* total,
                             uint64_t* false_positive);
/* Device-pointer forms (async on the context stream; smoothing synchronises
 * once to validate): confusion5 = tp, fp, tn, fn, exact; episodes3 =
 * detected, total, false_positive (device uint64, either nullable). */
hv_status hv_dev_smooth_labels(hv_context* ctx, const int32_t* labels, size_t n, size_t window, int32_t* out);
hv_status hv_dev_eval_counts(hv_context* ctx, const int32_t* pred, const int32_t* truth, size_t n,
                             int positive_class, uint64_t* confusion5, uint64_t* episodes3);

/* ---- HBM-resident experiment (run_experiment, experiment.cpp:280-345) ----
 * Folds of one resident dataset scatter their test predictions into a
 * device array (predicted[row], -1 = untested; a later fold overwrites);
 * finish concatenates the tested rows in original order, smooths binary runs
 * (class_count == 2 && smooth_window > 1, experiment.cpp:331-336), and scores
 * them (sample + episode metrics) without the predictions leaving HBM.
 * Outputs (host, nullable, capacity = dataset rows): tested row indices,
 * truth, raw prediction and final (smoothed) label per tested row. */
typedef struct hv_experiment hv_experiment;
hv_status hv_experiment_create(hv_context* ctx, const hv_dataset* ds, hv_experiment** out);
void hv_experiment_destroy(hv_experiment* ex);
hv_status hv_experiment_fold(hv_context* ctx, hv_experiment* ex, const uint64_t* train_idx, size_t n_train,
                             const uint64_t* test_idx, size_t n_test, size_t bins, const uint32_t* id_vectors,
                             const uint32_t* value_vectors, size_t dim, hv_binding binding,
                             const uint32_t* encode_tiebreak, size_t class_count, hv_metric metric, double gamma,
                             const uint32_t* model_tiebreak, int online, size_t batch_size);
hv_status hv_experiment_finish(hv_context* ctx, hv_experiment* ex, size_t class_count, size_t smooth_window,
                               int positive_class, hv_eval_report* report, uint64_t* n_tested,
                               uint64_t* tested_rows, int32_t* truth, int32_t* predicted, int32_t* final_labels);

/* model.hpp:67-70 hamming_distance / hamming_distance_words on the device:
 * popc(a ^ b) / dim in double (one row of the predict scan). */
hv_status hv_hamming_distance(hv_context* ctx, const uint32_t* a, const uint32_t* b, size_t dim, double* out);
/* model.hpp:74-75 cosine_similarity(acc, packed_row, dim): sequential fp64 dot
 * and norm like the reference; INVALID_ARGUMENT when acc_len != dim, DOMAIN
 * ("cosine_similarity: zero vector") for a zero accumulator or empty row. */
hv_status hv_cosine_similarity(hv_context* ctx, const double* acc, size_t acc_len, const uint32_t* row, size_t dim,
                               double* out);
/* model.hpp:67-70 hamming_distance_words (host-side helper, no device) */
double hv_hamming_distance_words(const uint32_t* a, const uint32_t* b, size_t dim);

/* Host-only (no device): narrow rows x features uint32 bins to uint8 rows of
 * pitch ldb (zero padded) on the library's host threads, as the host-pointer
 * calls do before their H2D copies; *first_bad = first flat index with a bin
 * >= bins, or UINT64_MAX. */
hv_status hv_host_narrow_bins(const uint32_t* bins32, size_t rows, size_t features, size_t bins,
                              uint8_t* out, size_t ldb, uint64_t* first_bad);

/* ---- device-resident API (device pointers, async on the context stream) -- */
/* Latched data errors of earlier hv_dev_* calls (synchronises the stream). */
hv_status hv_dev_check(hv_context* ctx);
/* uint32 bins (rows x features) -> validated uint8 bins with row pitch ldb >= features */
hv_status hv_dev_narrow_bins(hv_context* ctx, const uint32_t* bins32, size_t rows,
                             size_t features, size_t bins, uint8_t* bins8, size_t ldb);
/* Encode uint8 bins (row pitch ldb bytes) into rows x W words; bins already validated < bins.
 * Any binding; id-level takes the fused sm_100a path. */
hv_status hv_dev_encode(hv_context* ctx, const uint8_t* bins8, size_t ldb, size_t rows,
                        size_t features, const uint32_t* id_vectors,
                        const uint32_t* value_vectors, size_t bins, size_t dim,
                        hv_binding binding, const uint32_t* tiebreak, uint32_t* out);
/* Classical accumulation: counts (class_count x 32*W uint32, row-major) and
 * class_rows (class_count uint64) are ADDED to (zero them first); labels validated.
 * Sharded training calls this per shard and all-reduces counts/class_rows. */
hv_status hv_dev_class_counts(hv_context* ctx, const uint32_t* encoded, size_t rows, size_t dim,
                              const int32_t* labels, size_t class_count, uint32_t* counts,
                              uint64_t* class_rows);
/* Pitched hypervector rows (the engine's own HBM layout for resident data):
 * row r of an encoded matrix at encoded + r * ldw words, ldw >= W. With
 * ldw = hv_row_pitch_words(dim) (W rounded up to 16 bytes) and a 16-byte
 * aligned base, class counts stage whole rows with the bulk-copy engine and
 * predict reads uint4s; any other pitch takes the word-wise kernels. Words
 * [W, ldw) of a row are never read as data. hv_fold_* keep their rows so. */
size_t hv_row_pitch_words(size_t dim);
hv_status hv_dev_class_counts_pitched(hv_context* ctx, const uint32_t* encoded, size_t ldw, size_t rows,
                                      size_t dim, const int32_t* labels, size_t class_count,
                                      uint32_t* counts, uint64_t* class_rows);
/* Pitched predict: fewer than 32 classes (INVALID_ARGUMENT otherwise). */
hv_status hv_dev_predict_hamming_pitched(hv_context* ctx, const uint32_t* class_vectors,
                                         size_t class_count, size_t dim, const uint32_t* encoded,
                                         size_t ldw, size_t rows, int32_t* labels, double* distances,
                                         uint32_t* popcounts);
/* Binarise classical counts: bit = 2c > n ? 1 : 2c < n ? 0 : tiebreak. */
hv_status hv_dev_binarize_counts(hv_context* ctx, const uint32_t* counts,
                                 const uint64_t* class_rows, size_t class_count, size_t dim,
                                 const uint32_t* tiebreak, uint32_t* class_vectors);
/* Hamming nearest-class scan: labels (int32, nullable), distances (double rows x C,
 * nullable), popcounts (uint32 rows x C, nullable). */
hv_status hv_dev_predict_hamming(hv_context* ctx, const uint32_t* class_vectors,
                                 size_t class_count, size_t dim, const uint32_t* encoded,
                                 size_t rows, int32_t* labels, double* distances,
                                 uint32_t* popcounts);
/* Online training on device-resident state. acc: C x dim doubles, weight: C doubles,
 * counts: C uint64, class_vectors: C x W, tiebreak: 1 x W. Exact reference
 * semantics (sample-ordered in-place fp64 adds, snapshot per batch, bootstrap
 * batch visited twice). */
hv_status hv_dev_train_online(hv_context* ctx, const uint32_t* encoded, size_t rows, size_t dim,
                              const int32_t* labels, size_t class_count, size_t batch_size,
                              double gamma, const uint32_t* tiebreak, double* acc,
                              double* weight, uint64_t* counts, uint32_t* class_vectors);
/* One online batch in delta mode for data-parallel training: computes, against the
 * given (replicated) class vectors, this shard's per-class updates
 * delta_acc (C x dim, overwritten), delta_weight (C), delta_counts (C); the caller
 * all-reduces them and applies hv_dev_apply_online_delta. */
hv_status hv_dev_online_delta(hv_context* ctx, const uint32_t* class_vectors, size_t class_count,
                              size_t dim, const uint32_t* batch, size_t rows,
                              const int32_t* labels, double gamma, double* delta_acc,
                              double* delta_weight, uint64_t* delta_counts,
                              uint32_t* delta_touched);
/* acc += delta_acc; weight += delta_weight; counts += delta_counts; re-binarise the
 * classes with touched[c] != 0 (model.cpp:277-279). */
hv_status hv_dev_apply_online_delta(hv_context* ctx, size_t class_count, size_t dim,
                                    const double* delta_acc, const double* delta_weight,
                                    const uint64_t* delta_counts, const uint32_t* touched,
                                    const uint32_t* tiebreak, double* acc, double* weight,
                                    uint64_t* counts, uint32_t* class_vectors);
/* Encode only output words [word_begin, word_begin + word_count) of every row
 * into out (row stride ldo words) — the column slice a rank owns in D-sliced
 * training (encoding.cpp:266-271 is independent per output position). */
hv_status hv_dev_encode_words(hv_context* ctx, const uint8_t* bins8, size_t ldb, size_t rows,
                              size_t features, const uint32_t* id_vectors,
                              const uint32_t* value_vectors, size_t bins, size_t dim,
                              hv_binding binding, const uint32_t* tiebreak, size_t word_begin,
                              size_t word_count, uint32_t* out, size_t ldo);
/* ---- D-sliced exact online training (model.cpp:250-301 across ranks) -----
 * Rank r owns words [word_begin, word_begin + words) of every hypervector:
 * batch rows are its slice (row stride `words`), acc is C x slice_bits fp64
 * (slice_bits = min(dim, 32*(word_begin+words)) - 32*word_begin), class_vectors
 * C x words; weight/counts (C) are replicated and evolve identically.
 * Per batch: hv_dev_online_partial_popc -> all-reduce(sum) of popc (rows x C
 * uint32) -> hv_dev_online_slice_update. Every fp64 element sees the
 * reference's sample-ordered in-place additions: bit-identical to one GPU. */
hv_status hv_dev_online_slice_init(hv_context* ctx, const uint32_t* batch0, size_t rows0,
                                   const int32_t* labels, size_t class_count, size_t dim,
                                   size_t word_begin, size_t words, const uint32_t* tiebreak,
                                   double* acc, double* weight, uint64_t* counts,
                                   uint32_t* class_vectors);
hv_status hv_dev_online_partial_popc(hv_context* ctx, const uint32_t* class_vectors,
                                     size_t class_count, size_t words, const uint32_t* batch,
                                     size_t rows, uint32_t* popc);
/* hv_dev_online_partial_popc fused with the popcount all-reduce over peer
 * memory: ADDS this rank's partials into every rank's rows x C buffer
 * (peer_popc: device array of `world` device pointers, zeroed beforehand);
 * follow with hv_dev_signal_peers / hv_dev_wait_peers as for the counts. */
hv_status hv_dev_online_partial_popc_peers(hv_context* ctx, const uint32_t* class_vectors,
                                           size_t class_count, size_t words, const uint32_t* batch,
                                           size_t rows, uint32_t* const* peer_popc, size_t world);
/* Every batch of the word-sliced exact online mode, the popcount exchange
 * fused over peer memory, enqueued in one call: per batch the partial
 * popcounts are added into every rank's parity slot (peer_popc0/1: device
 * arrays of `world` slot pointers; own_popc0/1: this rank's), then signal /
 * wait on the flags (epochs epoch0+1 ..), score, lists and the slice update,
 * and this rank's slot is reset. State as hv_dev_online_slice_init left it. */
hv_status hv_dev_online_sliced_run_peers(hv_context* ctx, const uint32_t* enc_slice, size_t rows, size_t words,
                                         size_t word_begin, size_t dim, const int32_t* labels, size_t class_count,
                                         size_t batch_size, double gamma, const uint32_t* tiebreak,
                                         uint32_t* const* peer_popc0, uint32_t* const* peer_popc1, uint32_t* own_popc0,
                                         uint32_t* own_popc1, uint32_t* const* peer_flags, const uint32_t* own_flags,
                                         size_t world, size_t rank, uint32_t epoch0, double* acc, double* weight,
                                         uint64_t* counts, uint32_t* class_vectors);
hv_status hv_dev_online_slice_update(hv_context* ctx, const uint32_t* popc, size_t class_count,
                                     size_t dim, size_t word_begin, size_t words,
                                     const uint32_t* batch, size_t rows, const int32_t* labels,
                                     double gamma, const uint32_t* tiebreak, double* acc,
                                     double* weight, uint64_t* counts, uint32_t* class_vectors);
/* ---- classical training fused with its all-reduce over peer memory -------
 * (replaces hv_dev_class_counts + an NCCL all-reduce.) Each
 * rank shares a device buffer with its peers through CUDA IPC: */
size_t hv_shared_handle_size(void);  /* bytes of an IPC handle (64) */
hv_status hv_shared_alloc(hv_context* ctx, size_t bytes, void** dev_ptr, uint8_t* handle);
hv_status hv_shared_open(hv_context* ctx, const uint8_t* handle, void** dev_ptr);
hv_status hv_shared_close(hv_context* ctx, void* dev_ptr);
hv_status hv_shared_free(hv_context* ctx, void* dev_ptr);
/* Count this rank's rows (like hv_dev_class_counts) and add the exact counts
 * and class row counts into EVERY rank's buffers: peer_counts / peer_class_rows
 * are DEVICE arrays of `world` device pointers (C x 32W uint32, C uint64). */
hv_status hv_dev_class_counts_peers(hv_context* ctx, const uint32_t* encoded, size_t rows, size_t dim,
                                    const int32_t* labels, size_t class_count,
                                    uint32_t* const* peer_counts, uint64_t* const* peer_class_rows,
                                    size_t world);
hv_status hv_dev_class_counts_peers_pitched(hv_context* ctx, const uint32_t* encoded, size_t ldw,
                                            size_t rows, size_t dim, const int32_t* labels,
                                            size_t class_count, uint32_t* const* peer_counts,
                                            uint64_t* const* peer_class_rows, size_t world);
/* After the counts: store `epoch` into flag[rank] of every rank (peer_flags:
 * device array of `world` pointers to each rank's `world` uint32 flags) ... */
hv_status hv_dev_signal_peers(hv_context* ctx, uint32_t* const* peer_flags, size_t world, size_t rank,
                              uint32_t epoch);
/* ... and wait (on the stream) until this rank's flags all reach `epoch`;
 * a peer missing for 20 s latches an error reported by hv_dev_check. */
hv_status hv_dev_wait_peers(hv_context* ctx, const uint32_t* flags, size_t world, uint32_t epoch);
/* Synthetic workload (include/hvb200_synth.h) generated on device for rows
 * [row0, row0+rows): bins8 (pitch ldb) and labels. */
hv_status hv_dev_synth(hv_context* ctx, uint64_t row0, size_t rows, size_t features,
                       size_t class_count, size_t bins, int label_kind, uint64_t seed,
                       uint8_t* bins8, size_t ldb, int32_t* labels);

#ifdef __cplusplus
}
#endif
#endif /* HVB200_H */
