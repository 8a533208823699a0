"""Python mirror of the reference `hypervec` hot-path API over libhvb200.

Same names, argument meaning and error behaviour as the reference C++ headers
(/root/reference/proj/include/hypervec/{bitmat,kernels,encoding,model}.hpp):
reference `std::invalid_argument` surfaces as `InvalidArgument` (a
ValueError), `std::domain_error` as `DomainError`. Host data are numpy
arrays in the reference layout; every compute call runs the sm_100a kernels
through the C ABI (include/hvb200.h) — there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from ._native import (BIND_APPENDING, BIND_ID_LEVEL, BIND_PERMUTATION, GEN_RANDOM, GEN_SANDWICH,
                      GEN_SCALE_RANDOM, METRIC_COSINE, METRIC_HAMMING, DomainError, InvalidArgument,
                      LogicError)

__all__ = [
    "PackedBitMatrix", "DenseBitMatrix", "pack", "unpack", "xor_bind", "rotate", "horizontal_sum", "transpose",
    "vertical_sum", "majority_binarize", "popcount_words", "hamming_words", "Discretizer", "fit_discretizer",
    "discretize", "discretize_matrix", "generate_random", "generate_scale_random", "generate_sandwich",
    "Codebook", "make_codebook", "encode", "encode_batch", "ModelConfig", "HDModel", "ModelSnapshot",
    "Prediction", "make_empty_model", "train_classical", "freeze", "online_update", "train_online", "predict",
    "hamming_distance", "hamming_distance_words", "splitmix64", "derive_seed", "GenerationStrategy",
    "BindingStrategy", "Metric", "InvalidArgument", "DomainError", "LogicError",
]


class GenerationStrategy:  # encoding.hpp:17
    kRandom, kScaleRandom, kSandwich = GEN_RANDOM, GEN_SCALE_RANDOM, GEN_SANDWICH


class BindingStrategy:  # encoding.hpp:18
    kIdLevel, kPermutation, kAppending = BIND_ID_LEVEL, BIND_PERMUTATION, BIND_APPENDING


class Metric:  # model.hpp:17
    kHamming, kCosine = METRIC_HAMMING, METRIC_COSINE


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _ctx():
    return N.context(0).handle


def words_per_row(dim: int) -> int:
    return (dim + 31) // 32


# ------------------------------------------------------------ bitmat.hpp --
class PackedBitMatrix:
    """rows x dim bits in ceil(dim/32) uint32 words per row, LSB first (bitmat.hpp:15-94)."""

    def __init__(self, rows: int = 0, dim: int = 0, words: np.ndarray | None = None):
        self.dim = int(dim)
        w = words_per_row(self.dim)
        if words is None:
            words = np.zeros((rows, w), dtype=np.uint32)
        words = np.ascontiguousarray(words, dtype=np.uint32).reshape(-1, w) if w else np.zeros((rows, 0), np.uint32)
        self.words = words

    @property
    def rows(self) -> int:
        return self.words.shape[0]

    def words_per_row(self) -> int:
        return words_per_row(self.dim)

    def bit(self, r: int, j: int) -> bool:
        return bool((int(self.words[r, j // 32]) >> (j % 32)) & 1)

    def padding_clean(self) -> bool:
        rem = self.dim % 32
        if rem == 0 or self.words.size == 0:
            return True
        return not np.any(self.words[:, -1] & np.uint32(~((1 << rem) - 1) & 0xFFFFFFFF))

    def row(self, i: int) -> np.ndarray:
        return self.words[i]

    def __eq__(self, other) -> bool:
        return isinstance(other, PackedBitMatrix) and self.dim == other.dim and np.array_equal(self.words, other.words)


class DenseBitMatrix:
    """Byte-per-bit interchange matrix (bitmat.hpp:96-136)."""

    def __init__(self, rows: int = 0, dim: int = 0, bits: np.ndarray | None = None):
        if bits is None:
            bits = np.zeros((rows, dim), dtype=np.uint8)
        self.bits = np.ascontiguousarray(bits, dtype=np.uint8).reshape(-1, dim) if dim else np.zeros((rows, 0), np.uint8)
        self.dim = int(dim)

    @property
    def rows(self) -> int:
        return self.bits.shape[0]

    def __eq__(self, other) -> bool:
        return isinstance(other, DenseBitMatrix) and self.dim == other.dim and np.array_equal(self.bits, other.bits)


# ----------------------------------------------------------- kernels.hpp --
def pack(d: DenseBitMatrix) -> PackedBitMatrix:
    out = PackedBitMatrix(d.rows, d.dim)
    N.check(N.lib().hv_pack(_ctx(), _p(d.bits), d.rows, d.dim, _p(out.words)))
    return out


def unpack(m: PackedBitMatrix) -> DenseBitMatrix:
    out = DenseBitMatrix(m.rows, m.dim)
    N.check(N.lib().hv_unpack(_ctx(), _p(m.words), m.rows, m.dim, _p(out.bits)))
    return out


def xor_bind(a: PackedBitMatrix, b: PackedBitMatrix) -> PackedBitMatrix:
    out = PackedBitMatrix(a.rows, a.dim)
    N.check(N.lib().hv_xor_bind(_ctx(), _p(a.words), a.rows, a.dim, _p(b.words), b.rows, b.dim, _p(out.words)))
    return out


def rotate(m: PackedBitMatrix, shift: int) -> PackedBitMatrix:
    out = PackedBitMatrix(m.rows, m.dim)
    N.check(N.lib().hv_rotate(_ctx(), _p(m.words), m.rows, m.dim, shift, _p(out.words)))
    return out


def horizontal_sum(m: PackedBitMatrix) -> np.ndarray:
    out = np.zeros(m.rows, np.uint64)
    N.check(N.lib().hv_horizontal_sum(_ctx(), _p(m.words), m.rows, m.dim, _p(out)))
    return out


def transpose(m: PackedBitMatrix) -> PackedBitMatrix:
    out = PackedBitMatrix(m.dim, m.rows)
    N.check(N.lib().hv_transpose(_ctx(), _p(m.words), m.rows, m.dim, _p(out.words)))
    return out


def vertical_sum(m: PackedBitMatrix) -> np.ndarray:
    out = np.zeros(m.dim, np.uint64)
    N.check(N.lib().hv_vertical_sum(_ctx(), _p(m.words), m.rows, m.dim, _p(out)))
    return out


def majority_binarize(counts, n: int, tiebreak: PackedBitMatrix) -> PackedBitMatrix:
    counts = np.ascontiguousarray(counts, dtype=np.uint64)
    out = PackedBitMatrix(1, counts.shape[0])
    N.check(N.lib().hv_majority_binarize(_ctx(), _p(counts), counts.shape[0], n, _p(tiebreak.words), tiebreak.rows,
                                         tiebreak.dim, _p(out.words)))
    return out


def popcount_words(words) -> int:
    return int(np.unpackbits(np.ascontiguousarray(words, np.uint32).view(np.uint8)).sum())


def hamming_words(a, b) -> int:
    return popcount_words(np.bitwise_xor(np.asarray(a, np.uint32), np.asarray(b, np.uint32)))


# ---------------------------------------------------------- encoding.hpp --
@dataclass
class Discretizer:
    min: np.ndarray
    max: np.ndarray
    bins: int = 2

    def feature_count(self) -> int:
        return len(self.min)


def fit_discretizer(data, rows: int, features: int, bins: int) -> Discretizer:
    data = np.ascontiguousarray(data, dtype=np.float64).reshape(-1)
    if rows and features and data.size != rows * features:
        raise InvalidArgument("fit_discretizer: data length does not match rows x features")
    mn = np.zeros(features)
    mx = np.zeros(features)
    N.check(N.lib().hv_fit_discretizer(_ctx(), _p(data), rows, features, bins, _p(mn), _p(mx)))
    return Discretizer(mn, mx, bins)


def discretize_matrix(data, rows: int, d: Discretizer) -> np.ndarray:
    data = np.ascontiguousarray(data, dtype=np.float64).reshape(-1)
    f = d.feature_count()
    if data.size != rows * f:
        raise InvalidArgument("discretize_matrix: data length does not match rows x features")
    out = np.zeros(rows * f, np.uint32)
    N.check(N.lib().hv_discretize_matrix(_ctx(), _p(data), rows, f, _p(np.ascontiguousarray(d.min, np.float64)),
                                         _p(np.ascontiguousarray(d.max, np.float64)), d.bins, _p(out)))
    return out


def discretize(x, d: Discretizer) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float64).reshape(-1)
    if x.size != d.feature_count():
        raise InvalidArgument(f"discretize: expected {d.feature_count()} features, got {x.size}")
    return discretize_matrix(x, 1, d)


def splitmix64(x: int) -> int:
    return int(N.lib().hv_splitmix64(x))


def derive_seed(seed: int, tag: int) -> int:
    return int(N.lib().hv_derive_seed(seed, tag))


def generate_random(count: int, dim: int, seed: int) -> PackedBitMatrix:
    out = PackedBitMatrix(count, dim)
    N.check(N.lib().hv_generate_random(count, dim, seed, _p(out.words)))
    return out


def generate_scale_random(bins: int, dim: int, seed: int) -> PackedBitMatrix:
    out = PackedBitMatrix(bins, dim)
    N.check(N.lib().hv_generate_scale_random(bins, dim, seed, _p(out.words)))
    return out


def generate_sandwich(bins: int, dim: int, seed: int) -> PackedBitMatrix:
    out = PackedBitMatrix(bins, dim)
    N.check(N.lib().hv_generate_sandwich(bins, dim, seed, _p(out.words)))
    return out


@dataclass
class Codebook:  # encoding.hpp:65-75
    id_vectors: PackedBitMatrix
    value_vectors: PackedBitMatrix
    generation: int = GEN_RANDOM
    binding: int = BIND_ID_LEVEL
    seed: int = 0

    def feature_count(self) -> int:
        return self.id_vectors.rows

    def bin_count(self) -> int:
        return self.value_vectors.rows

    def dim(self) -> int:
        return self.id_vectors.dim


def make_codebook(generation: int, binding: int, features: int, bins: int, dim: int, seed: int) -> Codebook:
    idv = PackedBitMatrix(features, dim)
    val = PackedBitMatrix(bins, dim)
    N.check(N.lib().hv_make_codebook(generation, features, bins, dim, seed, _p(idv.words), _p(val.words)))
    return Codebook(idv, val, generation, binding, seed)


def encode_batch(bin_rows, rows: int, codebook: Codebook, tiebreak: PackedBitMatrix, threads: int = 1) -> PackedBitMatrix:
    """encoding.hpp:91-93; `threads` is accepted for API parity (the GPU ignores it)."""
    f = codebook.feature_count()
    bin_rows = np.ascontiguousarray(bin_rows, dtype=np.uint32).reshape(-1)
    if bin_rows.size != rows * f:
        raise InvalidArgument("encode_batch: bin matrix length does not match rows x features")
    out = PackedBitMatrix(rows, codebook.dim())
    N.check(N.lib().hv_encode_batch(_ctx(), _p(bin_rows), rows, f, _p(codebook.id_vectors.words),
                                    _p(codebook.value_vectors.words), codebook.bin_count(), codebook.dim(),
                                    codebook.binding, _p(tiebreak.words), tiebreak.rows, tiebreak.dim,
                                    _p(out.words)))
    return out


def encode(bins, codebook: Codebook, tiebreak: PackedBitMatrix) -> PackedBitMatrix:
    bins = np.ascontiguousarray(bins, dtype=np.uint32).reshape(-1)
    if bins.size != codebook.feature_count():
        raise InvalidArgument(f"encode: expected {codebook.feature_count()} bin indices, got {bins.size}")
    return encode_batch(bins, 1, codebook, tiebreak)


# ------------------------------------------------------------- model.hpp --
@dataclass
class ModelConfig:  # model.hpp:22-28
    class_count: int = 2
    dim: int = 0
    metric: int = METRIC_HAMMING
    gamma: float = 1.0
    seed: int = 1


@dataclass
class HDModel:  # model.hpp:37-56
    config: ModelConfig
    accumulators: np.ndarray
    class_weight: np.ndarray
    sample_counts: np.ndarray
    class_vectors: PackedBitMatrix
    tiebreak: PackedBitMatrix

    @classmethod
    def allocate(cls, cfg: ModelConfig) -> "HDModel":
        c, d = cfg.class_count, cfg.dim
        return cls(ModelConfig(**vars(cfg)), np.zeros(c * d), np.zeros(c), np.zeros(c, np.uint64),
                   PackedBitMatrix(c, d), PackedBitMatrix(1, d))

    def _struct(self) -> N.Model:
        cfg = self.config
        return N.Model(cfg.class_count, cfg.dim, cfg.metric, cfg.gamma, cfg.seed, self.accumulators.ctypes.data,
                       self.class_weight.ctypes.data, self.sample_counts.ctypes.data,
                       self.class_vectors.words.ctypes.data, self.tiebreak.words.ctypes.data)

    def accumulator_row(self, c: int) -> np.ndarray:
        d = self.config.dim
        return self.accumulators[c * d:(c + 1) * d]

    def class_empty(self, c: int) -> bool:
        return int(self.sample_counts[c]) == 0

    def refresh_binarization(self, c: int | None = None) -> None:
        s = self._struct()
        N.check(N.lib().hv_refresh_binarization(_ctx(), C.byref(s), (1 << 64) - 1 if c is None else c))


@dataclass
class ModelSnapshot:  # model.hpp:86-89
    class_vectors: PackedBitMatrix
    accumulators: np.ndarray


@dataclass
class Prediction:  # model.hpp:61-64
    label: int
    distances: np.ndarray = field(default_factory=lambda: np.zeros(0))


def _check_cfg(cfg: ModelConfig):
    if cfg.class_count == 0:
        raise InvalidArgument("make_empty_model: need at least one class")


def make_empty_model(cfg: ModelConfig) -> HDModel:
    if cfg.class_count == 0:
        raise InvalidArgument("make_empty_model: need at least one class")
    if cfg.dim == 0:
        raise InvalidArgument("make_empty_model: dim must be >= 1")
    m = HDModel.allocate(cfg)
    s = m._struct()
    N.check(N.lib().hv_make_empty_model(C.byref(s)))
    return m


def _labels(labels) -> np.ndarray:
    return np.ascontiguousarray(labels, dtype=np.int32).reshape(-1)


def train_classical(encoded: PackedBitMatrix, labels, config: ModelConfig) -> HDModel:
    y = _labels(labels)
    cfg = ModelConfig(**vars(config))
    cfg.dim = encoded.dim
    m = HDModel.allocate(cfg) if cfg.class_count and cfg.dim else HDModel.allocate(ModelConfig(max(cfg.class_count, 1), max(cfg.dim, 1)))
    m.config = cfg
    s = m._struct()
    N.check(N.lib().hv_train_classical(_ctx(), _p(encoded.words), encoded.rows, encoded.dim, _p(y), y.size,
                                       C.byref(s)))
    return m


def freeze(model: HDModel) -> ModelSnapshot:
    return ModelSnapshot(PackedBitMatrix(model.class_vectors.rows, model.class_vectors.dim,
                                         model.class_vectors.words.copy()), model.accumulators.copy())


def online_update(model: HDModel, batch: PackedBitMatrix, labels, frozen: ModelSnapshot) -> None:
    y = _labels(labels)
    s = model._struct()
    acc = frozen.accumulators if model.config.metric == METRIC_COSINE else None
    N.check(N.lib().hv_online_update(_ctx(), C.byref(s), _p(batch.words), batch.rows, batch.dim, _p(y), y.size,
                                     _p(frozen.class_vectors.words), _p(acc)))


def train_online(encoded: PackedBitMatrix, labels, batch_size: int, config: ModelConfig) -> HDModel:
    y = _labels(labels)
    cfg = ModelConfig(**vars(config))
    cfg.dim = encoded.dim
    m = HDModel.allocate(cfg) if cfg.class_count and cfg.dim else HDModel.allocate(ModelConfig(max(cfg.class_count, 1), max(cfg.dim, 1)))
    m.config = cfg
    s = m._struct()
    N.check(N.lib().hv_train_online(_ctx(), _p(encoded.words), encoded.rows, encoded.dim, _p(y), y.size, batch_size,
                                    C.byref(s)))
    return m


def predict(model: HDModel, encoded: PackedBitMatrix, threads: int = 1) -> list[Prediction]:
    labels, dist = predict_arrays(model, encoded)
    return [Prediction(int(labels[i]), dist[i]) for i in range(encoded.rows)]


def predict_arrays(model: HDModel, encoded: PackedBitMatrix, distances: bool = True):
    """Vectorised predict: (labels int32[rows], distances float64[rows, C] or None)."""
    labels = np.zeros(encoded.rows, np.int32)
    dist = np.zeros((encoded.rows, model.config.class_count)) if distances else None
    s = model._struct()
    N.check(N.lib().hv_predict(_ctx(), C.byref(s), _p(encoded.words), encoded.rows, encoded.dim, _p(labels), _p(dist)))
    return labels, dist


def hamming_distance_words(a, b, dim: int) -> float:
    """model.cpp:178-181 on the device (one row of the predict scan)."""
    a = np.ascontiguousarray(a, np.uint32)
    b = np.ascontiguousarray(b, np.uint32)
    out = C.c_double()
    N.check(N.lib().hv_hamming_distance(_ctx(), _p(a), _p(b), dim, C.byref(out)))
    return out.value


def cosine_similarity(acc, packed_row, dim: int) -> float:
    """model.cpp:183-196: cosine of an accumulator row against a packed row
    (sequential fp64 like the reference); DomainError on a zero vector."""
    acc = np.ascontiguousarray(acc, np.float64)
    row = np.ascontiguousarray(packed_row, np.uint32)
    out = C.c_double()
    N.check(N.lib().hv_cosine_similarity(_ctx(), _p(acc), acc.size, _p(row), dim, C.byref(out)))
    return out.value


def hamming_distance(a: PackedBitMatrix, row_a: int, b: PackedBitMatrix, row_b: int) -> float:
    if a.dim != b.dim:
        raise InvalidArgument(f"hamming_distance: dimensions {a.dim} vs {b.dim}")
    return hamming_distance_words(a.words[row_a], b.words[row_b], a.dim)


@dataclass
class EpisodeCounts:  # eval.hpp:13-17
    detected: int = 0
    total: int = 0
    false_positive: int = 0


@dataclass
class EvalReport:
    """eval.hpp:26-37: absent ratios are None (the reference's std::nullopt)."""

    tp: int = 0
    fp: int = 0
    tn: int = 0
    fn: int = 0
    accuracy: float = 0.0
    tpr: float | None = None
    ppv: float | None = None
    f1: float | None = None
    episodes: EpisodeCounts | None = None

    @classmethod
    def _from_c(cls, r: "N.EvalReportC", episodes: bool) -> "EvalReport":
        return cls(int(r.tp), int(r.fp), int(r.tn), int(r.fn), r.accuracy, r.tpr if r.has_tpr else None,
                   r.ppv if r.has_ppv else None, r.f1 if r.has_f1 else None,
                   EpisodeCounts(int(r.episodes_detected), int(r.episodes_total), int(r.episodes_false_positive))
                   if episodes else None)


def smooth_labels(labels, window: int) -> np.ndarray:
    """eval.cpp:12-37 on the device (prefix-count scan + windowed majority)."""
    a = np.ascontiguousarray(labels, np.int32)
    out = np.zeros(max(a.size, 1), np.int32)
    N.check(N.lib().hv_smooth_labels(_ctx(), _p(a), a.size, window, _p(out)))
    return out[:a.size]


def sample_metrics(pred, truth, positive_class: int) -> EvalReport:
    """eval.cpp:39-77: confusion counts on the device, ratios as the reference forms them."""
    p = np.ascontiguousarray(pred, np.int32)
    t = np.ascontiguousarray(truth, np.int32)
    r = N.EvalReportC()
    N.check(N.lib().hv_sample_metrics(_ctx(), _p(p), p.size, _p(t), t.size, positive_class, C.byref(r)))
    return EvalReport._from_c(r, episodes=False)


def episode_metrics(pred, truth, positive_class: int) -> EpisodeCounts:
    """eval.cpp:79-116: run-level detection counts (one device scan)."""
    p = np.ascontiguousarray(pred, np.int32)
    t = np.ascontiguousarray(truth, np.int32)
    d, n, f = C.c_uint64(), C.c_uint64(), C.c_uint64()
    N.check(N.lib().hv_episode_metrics(_ctx(), _p(p), p.size, _p(t), t.size, positive_class, C.byref(d),
                                       C.byref(n), C.byref(f)))
    return EpisodeCounts(d.value, n.value, f.value)


class Dataset:
    """An HBM-resident feature matrix for repeated folds (run_fold_packed,
    experiment.cpp:148-178, with the discretizer re-fit per fold on device)."""

    def __init__(self, X, labels):
        X = np.ascontiguousarray(X, np.float64)
        y = np.ascontiguousarray(labels, np.int32)
        if X.ndim != 2 or y.shape[0] != X.shape[0]:
            raise InvalidArgument("dataset: X must be rows x features with one label per row")
        self.rows, self.features = X.shape
        h = C.c_void_p()
        N.check(N.lib().hv_dataset_create(_ctx(), _p(X), self.rows, self.features, _p(y), C.byref(h)))
        self._h = h

    def fold(self, train_idx, test_idx, codebook: Codebook, encode_tiebreak: PackedBitMatrix, cfg: ModelConfig,
             trainer: str = "classical", batch_size: int = 1024):
        """Labels of the test rows, plus the fitted (min, max) of the train rows."""
        tr = np.ascontiguousarray(train_idx, np.uint64)
        te = np.ascontiguousarray(test_idx, np.uint64)
        labels = np.zeros(max(te.size, 1), np.int32)
        mn = np.zeros(self.features)
        mx = np.zeros(self.features)
        mtb = PackedBitMatrix(1, cfg.dim)
        N.check(N.lib().hv_generate_random(1, cfg.dim, N.lib().hv_derive_seed(cfg.seed, 3), _p(mtb.words)))
        N.check(N.lib().hv_dataset_fold(_ctx(), self._h, _p(tr), tr.size, _p(te), te.size,
                                        codebook.bin_count(), _p(codebook.id_vectors.words),
                                        _p(codebook.value_vectors.words), cfg.dim, codebook.binding,
                                        _p(encode_tiebreak.words), cfg.class_count, cfg.metric, cfg.gamma,
                                        _p(mtb.words), 1 if trainer == "online" else 0, batch_size, _p(labels),
                                        _p(mn), _p(mx)))
        return labels[:te.size], mn, mx

    def experiment(self) -> "Experiment":
        return Experiment(self)

    def close(self):
        if self._h:
            N.lib().hv_dataset_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class ExperimentResult:
    """experiment.hpp ExperimentResult / PredictionRow columns, as arrays."""

    fold_count: int
    report: EvalReport
    rows: np.ndarray       # tested row indices, original order
    truth: np.ndarray
    predicted: np.ndarray  # raw fold predictions
    final: np.ndarray      # after smoothing


class Experiment:
    """run_experiment (experiment.cpp:280-345) over an HBM-resident Dataset:
    every fold scatters its predictions on device; finish() concatenates the
    tested rows, smooths binary runs and scores them without a host round trip."""

    def __init__(self, ds: Dataset):
        self.ds = ds
        self.folds = 0
        h = C.c_void_p()
        N.check(N.lib().hv_experiment_create(_ctx(), ds._h, C.byref(h)))
        self._h = h

    def fold(self, train_idx, test_idx, codebook: Codebook, encode_tiebreak: PackedBitMatrix, cfg: ModelConfig,
             trainer: str = "classical", batch_size: int = 1024):
        tr = np.ascontiguousarray(train_idx, np.uint64)
        te = np.ascontiguousarray(test_idx, np.uint64)
        mtb = PackedBitMatrix(1, cfg.dim)
        N.check(N.lib().hv_generate_random(1, cfg.dim, N.lib().hv_derive_seed(cfg.seed, 3), _p(mtb.words)))
        N.check(N.lib().hv_experiment_fold(_ctx(), self._h, _p(tr), tr.size, _p(te), te.size,
                                           codebook.bin_count(), _p(codebook.id_vectors.words),
                                           _p(codebook.value_vectors.words), cfg.dim, codebook.binding,
                                           _p(encode_tiebreak.words), cfg.class_count, cfg.metric, cfg.gamma,
                                           _p(mtb.words), 1 if trainer == "online" else 0, batch_size))
        self.folds += 1

    def finish(self, class_count: int, smooth_window: int = 1, positive_class: int = 1) -> ExperimentResult:
        rows = self.ds.rows
        r = N.EvalReportC()
        m = C.c_uint64()
        idx = np.zeros(max(rows, 1), np.uint64)
        truth, pred, fin = (np.zeros(max(rows, 1), np.int32) for _ in range(3))
        N.check(N.lib().hv_experiment_finish(_ctx(), self._h, class_count, smooth_window, positive_class,
                                             C.byref(r), C.byref(m), _p(idx), _p(truth), _p(pred), _p(fin)))
        k = m.value
        return ExperimentResult(self.folds, EvalReport._from_c(r, episodes=True), idx[:k], truth[:k], pred[:k],
                                fin[:k])

    def close(self):
        if self._h:
            N.lib().hv_experiment_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
