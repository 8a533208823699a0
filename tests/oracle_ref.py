"""ctypes view of the C oracle (oracle/liboracle.so) — test infrastructure only.

The oracle restates the reference's hot path on the CPU (oracle/hv_oracle.c,
each function citing /root/reference/proj file:line). Tests use it as the
checker for the CUDA engine; it is pinned against the reference's own golden
vectors in tests/test_oracle_golden.py.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
_LIB_PATH = ROOT / "oracle" / "liboracle.so"

HAMMING, COSINE = 0, 1
GEN_RANDOM, GEN_SCALE_RANDOM, GEN_SANDWICH = 0, 1, 2
BIND_ID_LEVEL, BIND_PERMUTATION, BIND_APPENDING = 0, 1, 2

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            import subprocess

            subprocess.run(["make", "-C", str(ROOT / "oracle"), "liboracle.so"], check=True,
                           stdout=subprocess.DEVNULL)
        _lib = C.CDLL(str(_LIB_PATH))
        _declare(_lib)
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def _declare(L):
    sz, u64, vp = C.c_size_t, C.c_uint64, C.c_void_p
    L.hvo_splitmix64.restype = u64
    L.hvo_splitmix64.argtypes = [u64]
    L.hvo_derive_seed.restype = u64
    L.hvo_derive_seed.argtypes = [u64, u64]
    L.hvo_mt64_stream.argtypes = [u64, sz, vp]
    L.hvo_generate_random.argtypes = [sz, sz, u64, vp]
    L.hvo_generate_scale_random.argtypes = [sz, sz, u64, vp]
    L.hvo_generate_sandwich.argtypes = [sz, sz, u64, vp]
    L.hvo_make_codebook.argtypes = [C.c_int, sz, sz, sz, u64, vp, vp]
    L.hvo_pack.restype = C.c_longlong
    L.hvo_pack.argtypes = [vp, sz, sz, vp]
    L.hvo_unpack.argtypes = [vp, sz, sz, vp]
    L.hvo_xor_bind.argtypes = [vp, sz, vp, sz, sz, vp]
    L.hvo_rotate.argtypes = [vp, sz, sz, sz, vp]
    L.hvo_horizontal_sum.argtypes = [vp, sz, sz, vp]
    L.hvo_transpose.argtypes = [vp, sz, sz, vp]
    L.hvo_vertical_sum.argtypes = [vp, sz, sz, vp]
    L.hvo_majority_binarize.restype = C.c_longlong
    L.hvo_majority_binarize.argtypes = [vp, sz, u64, vp, vp]
    L.hvo_fit_discretizer.argtypes = [vp, sz, sz, sz, vp, vp]
    L.hvo_discretize_matrix.argtypes = [vp, sz, sz, vp, vp, sz, vp]
    L.hvo_encode_batch.argtypes = [vp, sz, sz, vp, vp, sz, sz, C.c_int, vp, vp, vp]
    for name in ("hvo_train_classical", "hvo_online_update", "hvo_train_online", "hvo_predict"):
        getattr(L, name).restype = C.c_int


# ---------------------------------------------------------------- packing --
def _declare_eval(L):
    sz, vp = C.c_size_t, C.c_void_p
    L.hvo_smooth_labels.argtypes = [vp, sz, sz, vp, vp]
    L.hvo_sample_metrics.argtypes = [vp, sz, vp, sz, C.c_int, vp, vp]
    L.hvo_episode_metrics.argtypes = [vp, sz, vp, sz, C.c_int, vp]


def smooth_labels(labels, window):
    """eval.cpp:12-37 via hvo_smooth_labels; ValueError like the reference's invalid_argument."""
    L = lib()
    _declare_eval(L)
    a = np.ascontiguousarray(labels, np.int32)
    out = np.zeros(len(a), np.int32)
    bad = np.zeros(1, np.uint64)
    if L.hvo_smooth_labels(_p(a), len(a), window, _p(out), _p(bad)) != 0:
        raise ValueError(f"smooth_labels: bad input at {int(bad[0])}")
    return out


def sample_metrics(pred, truth, positive):
    """eval.cpp:39-77 -> (counts[tp, fp, tn, fn, exact], ratios[acc, tpr, ppv, f1]; NaN = absent)."""
    L = lib()
    _declare_eval(L)
    p, t = np.ascontiguousarray(pred, np.int32), np.ascontiguousarray(truth, np.int32)
    counts, ratios = np.zeros(5, np.uint64), np.zeros(4, np.float64)
    if L.hvo_sample_metrics(_p(p), len(p), _p(t), len(t), positive, _p(counts), _p(ratios)) != 0:
        raise ValueError("sample_metrics: bad input")
    return counts, ratios


def episode_metrics(pred, truth, positive):
    """eval.cpp:79-116 -> [detected, total, false_positive]."""
    L = lib()
    _declare_eval(L)
    p, t = np.ascontiguousarray(pred, np.int32), np.ascontiguousarray(truth, np.int32)
    out = np.zeros(3, np.uint64)
    if L.hvo_episode_metrics(_p(p), len(p), _p(t), len(t), positive, _p(out)) != 0:
        raise ValueError("episode_metrics: bad input")
    return out


def words_per_row(dim: int) -> int:
    return (dim + 31) // 32


def pack_rows(dense: np.ndarray) -> np.ndarray:
    """(n, D) 0/1 uint8 -> (n, ceil(D/32)) uint32, LSB-first (bitmat.hpp:15-19)."""
    dense = np.ascontiguousarray(dense, dtype=np.uint8)
    n, d = dense.shape
    w = words_per_row(d)
    b = np.packbits(dense, axis=1, bitorder="little")
    out = np.zeros((n, 4 * w), dtype=np.uint8)
    out[:, : b.shape[1]] = b
    return out.view("<u4").reshape(n, w).copy()


def unpack_rows(words: np.ndarray, dim: int) -> np.ndarray:
    words = np.ascontiguousarray(words, dtype="<u4")
    n = words.shape[0]
    bits = np.unpackbits(words.view(np.uint8).reshape(n, -1), axis=1, bitorder="little")
    return bits[:, :dim].copy()


# ------------------------------------------------------------------ rng ----
def mt64(seed: int, n: int) -> np.ndarray:
    out = np.zeros(n, dtype=np.uint64)
    lib().hvo_mt64_stream(seed, n, _p(out))
    return out


def derive_seed(seed: int, tag: int) -> int:
    return int(lib().hvo_derive_seed(seed, tag))


def splitmix64(x: int) -> int:
    return int(lib().hvo_splitmix64(x))


def generate_random(count: int, dim: int, seed: int) -> np.ndarray:
    out = np.zeros((count, words_per_row(dim)), dtype=np.uint32)
    lib().hvo_generate_random(count, dim, seed, _p(out))
    return out


def generate_scale_random(bins: int, dim: int, seed: int) -> np.ndarray:
    out = np.zeros((bins, words_per_row(dim)), dtype=np.uint32)
    if lib().hvo_generate_scale_random(bins, dim, seed, _p(out)) != 0:
        raise ValueError("generate_scale_random: invalid argument")
    return out


def generate_sandwich(bins: int, dim: int, seed: int) -> np.ndarray:
    out = np.zeros((bins, words_per_row(dim)), dtype=np.uint32)
    if lib().hvo_generate_sandwich(bins, dim, seed, _p(out)) != 0:
        raise ValueError("generate_sandwich: invalid argument")
    return out


def make_codebook(generation: int, features: int, bins: int, dim: int, seed: int):
    w = words_per_row(dim)
    idv = np.zeros((features, w), dtype=np.uint32)
    val = np.zeros((bins, w), dtype=np.uint32)
    if lib().hvo_make_codebook(generation, features, bins, dim, seed, _p(idv), _p(val)) != 0:
        raise ValueError("make_codebook: invalid argument")
    return idv, val


# -------------------------------------------------------------- kernels ----
def xor_bind(a, b):
    a = np.ascontiguousarray(a, np.uint8)
    b = np.ascontiguousarray(b, np.uint8)
    out = np.zeros_like(a)
    assert lib().hvo_xor_bind(_p(a), a.shape[0], _p(b), b.shape[0], a.shape[1], _p(out)) == 0
    return out


def rotate(m, shift):
    m = np.ascontiguousarray(m, np.uint8)
    out = np.zeros_like(m)
    lib().hvo_rotate(_p(m), m.shape[0], m.shape[1], shift, _p(out))
    return out


def horizontal_sum(m):
    m = np.ascontiguousarray(m, np.uint8)
    out = np.zeros(m.shape[0], np.uint64)
    lib().hvo_horizontal_sum(_p(m), m.shape[0], m.shape[1], _p(out))
    return out


def transpose(m):
    m = np.ascontiguousarray(m, np.uint8)
    out = np.zeros((m.shape[1], m.shape[0]), np.uint8)
    lib().hvo_transpose(_p(m), m.shape[0], m.shape[1], _p(out))
    return out


def vertical_sum(m):
    m = np.ascontiguousarray(m, np.uint8)
    out = np.zeros(m.shape[1], np.uint64)
    lib().hvo_vertical_sum(_p(m), m.shape[0], m.shape[1], _p(out))
    return out


def majority_binarize(counts, n, tiebreak):
    counts = np.ascontiguousarray(counts, np.uint64)
    tiebreak = np.ascontiguousarray(tiebreak, np.uint8).reshape(-1)
    out = np.zeros(counts.shape[0], np.uint8)
    bad = lib().hvo_majority_binarize(_p(counts), counts.shape[0], n, _p(tiebreak), _p(out))
    if bad >= 0:
        raise ValueError(f"majority_binarize: count exceeds total at position {bad}")
    return out


def fit_discretizer(data, bins):
    data = np.ascontiguousarray(data, np.float64)
    rows, feats = data.shape
    mn = np.zeros(feats)
    mx = np.zeros(feats)
    if lib().hvo_fit_discretizer(_p(data), rows, feats, bins, _p(mn), _p(mx)) != 0:
        raise ValueError("fit_discretizer: invalid argument")
    return mn, mx


def discretize_matrix(data, mn, mx, bins):
    data = np.ascontiguousarray(data, np.float64)
    out = np.zeros(data.shape, np.uint32)
    lib().hvo_discretize_matrix(_p(data), data.shape[0], data.shape[1], _p(np.ascontiguousarray(mn)),
                                _p(np.ascontiguousarray(mx)), bins, _p(out))
    return out


def encode_batch(bins, id_words, value_words, n_bins, dim, binding, tiebreak_words):
    """Packed codebook in, packed HVs out; computed byte-per-bit (reference.cpp:202-267)."""
    bins = np.ascontiguousarray(bins, np.uint32)
    rows, feats = bins.shape
    idd = unpack_rows(id_words, dim)
    vd = unpack_rows(value_words, dim)
    tb = unpack_rows(np.asarray(tiebreak_words).reshape(1, -1), dim)
    out = np.zeros((rows, dim), np.uint8)
    bad = C.c_longlong(-1)
    st = lib().hvo_encode_batch(_p(bins), rows, feats, _p(idd), _p(vd), n_bins, dim, binding,
                                _p(tb), _p(out), C.byref(bad))
    if st != 0:
        raise ValueError(f"encode: invalid argument (flat index {bad.value})")
    return pack_rows(out)


# ---------------------------------------------------------------- model ----
class _Model(C.Structure):
    _fields_ = [("class_count", C.c_size_t), ("dim", C.c_size_t), ("metric", C.c_int),
                ("gamma", C.c_double), ("accumulators", C.c_void_p), ("class_weight", C.c_void_p),
                ("sample_counts", C.c_void_p), ("class_vectors", C.c_void_p), ("tiebreak", C.c_void_p)]


class NaiveModel:
    """Byte-per-bit model mirror (reference.hpp:43-54)."""

    def __init__(self, classes, dim, tiebreak_words, metric=HAMMING, gamma=1.0):
        self.classes, self.dim, self.metric, self.gamma = classes, dim, metric, gamma
        self.acc = np.zeros((classes, dim), np.float64)
        self.weight = np.zeros(classes, np.float64)
        self.counts = np.zeros(classes, np.uint64)
        self.cv = np.zeros((classes, dim), np.uint8)
        self.tiebreak = unpack_rows(np.asarray(tiebreak_words).reshape(1, -1), dim).reshape(-1).copy()

    def _s(self):
        return _Model(self.classes, self.dim, self.metric, self.gamma, self.acc.ctypes.data,
                      self.weight.ctypes.data, self.counts.ctypes.data, self.cv.ctypes.data,
                      self.tiebreak.ctypes.data)

    @property
    def class_vectors(self):
        return pack_rows(self.cv)

    def train_classical(self, enc_words, labels):
        e = unpack_rows(enc_words, self.dim)
        y = np.ascontiguousarray(labels, np.int32)
        s = self._s()
        assert lib().hvo_train_classical(C.byref(s), _p(e), e.shape[0], _p(y)) == 0
        return self

    def online_update(self, batch_words, labels):
        e = unpack_rows(batch_words, self.dim)
        y = np.ascontiguousarray(labels, np.int32)
        snap_cv = self.cv.copy()
        snap_acc = self.acc.copy()
        s = self._s()
        st = lib().hvo_online_update(C.byref(s), _p(e), e.shape[0], _p(y), _p(snap_cv), _p(snap_acc))
        assert st == 0, st
        return self

    def train_online(self, enc_words, labels, batch_size):
        e = unpack_rows(enc_words, self.dim)
        y = np.ascontiguousarray(labels, np.int32)
        s = self._s()
        assert lib().hvo_train_online(C.byref(s), _p(e), e.shape[0], _p(y), batch_size) == 0
        return self

    def predict(self, enc_words):
        e = unpack_rows(enc_words, self.dim)
        labels = np.zeros(e.shape[0], np.int32)
        dist = np.zeros((e.shape[0], self.classes), np.float64)
        s = self._s()
        st = lib().hvo_predict(C.byref(s), _p(e), e.shape[0], _p(labels), _p(dist))
        if st == 2:
            raise ArithmeticError("cosine_similarity: zero query vector")
        assert st == 0
        return labels, dist


def synth_bins(rows, features, classes, bins, seed, label_kind, start=0):
    """Python restatement of include/hvb200_synth.h (vectorised, for tests)."""
    M64 = (1 << 64) - 1
    i = np.arange(start, start + rows, dtype=np.uint64)
    if label_kind == 1:
        y = ((i % np.uint64(40000)) < np.uint64(120)).astype(np.int32)
    else:
        y = (i % np.uint64(classes)).astype(np.int32)
    f = np.arange(features, dtype=np.uint64)
    centre = ((y.astype(np.uint64)[:, None] * (f[None, :] + np.uint64(1)) + np.uint64(3) * f[None, :])
              % np.uint64(16)) % np.uint64(bins)
    with np.errstate(over="ignore"):
        ctr = (i[:, None] * np.uint64(features) + f[None, :]) * np.uint64(0xD6E8FEB86659FD93)
        x = np.uint64(seed) ^ ctr
        x = x + np.uint64(0x9E3779B97F4A7C15)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        x = x ^ (x >> np.uint64(31))
    u = (x >> np.uint64(61)).astype(np.int64)
    c = centre.astype(np.int64)
    out = np.where((u == 0) & (c > 0), c - 1, np.where((u == 1) & (c + 1 < bins), c + 1, c))
    del M64
    return out.astype(np.uint32), y


def make_synth(rows, features, classes, seed, grid_bins=16, jitter=0.3):
    """Reference test-support make_synth (tests/support/synth.cpp:16-47) via
    the oracle's C restatement: fp64 features (rows x features) and labels."""
    L = lib()
    L.hvo_make_synth.restype = C.c_int
    L.hvo_make_synth.argtypes = [C.c_size_t, C.c_size_t, C.c_size_t, C.c_size_t, C.c_double, C.c_uint64,
                                 C.c_void_p, C.c_void_p]
    X = np.zeros((rows, features), np.float64)
    y = np.zeros(rows, np.int32)
    assert L.hvo_make_synth(rows, features, classes, grid_bins, jitter, seed, _p(X), _p(y)) == 0
    return X, y


def fnv_rows(a):
    """FNV-1a 64 of each row of a 2-D uint32 / float64 array (oracle/golden_gen.cpp
    fnv_words / fnv_doubles): the digests the big golden pipelines store."""
    a = np.ascontiguousarray(a)
    v = a.view(np.uint64) if a.dtype == np.float64 else a.astype(np.uint64)
    h = np.full(v.shape[0], 1469598103934665603, np.uint64)
    with np.errstate(over="ignore"):
        for j in range(v.shape[1]):
            h = (h ^ v[:, j]) * np.uint64(1099511628211)
    return h


def synth_c(row0, rows, features, classes, bins, kind, seed):
    """The C generator (include/hvb200_synth.h) via the oracle library."""
    L = lib()
    L.hvo_synth.argtypes = [C.c_uint64, C.c_size_t, C.c_size_t, C.c_size_t, C.c_size_t, C.c_int, C.c_uint64,
                            C.c_void_p, C.c_void_p]
    b = np.zeros((rows, features), np.uint32)
    y = np.zeros(rows, np.int32)
    L.hvo_synth(row0, rows, features, classes, bins, kind, seed, _p(b), _p(y))
    return b, y
