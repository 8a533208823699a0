"""Binary containers of the reference, byte for byte.

Host-side serialisation of what the engine produces, so that hypervectors,
codebooks and models written here are byte-identical to the reference's and
load in either direction:

* ``HVPB`` packed bit matrix — io.cpp:85-107 (magic, u16 version, u64 rows,
  u64 dim, LE u32 words; a reader rejects set padding bits);
* ``HVCB`` codebook — encoding.cpp:313-363 (magic, u16 version, u64 JSON
  length, compact JSON header with sorted keys, then the ID and value
  matrices as HVPB);
* ``HVMD`` model — model.cpp:322-372 (magic, version, JSON header, class
  vectors as HVPB, then accumulators f64, class weights f64, sample counts
  u64, all little endian).

The JSON headers are nlohmann::json ``dump()`` output (keys sorted, no
spaces); doubles use its shortest-round-trip format (``_json_double``).
Errors are ``RuntimeError`` with the reference's messages (std::runtime_error).
"""
from __future__ import annotations

import decimal
import io as _io
import json
import struct

import numpy as np

from . import hypervec as hv

VERSION = 1  # io.hpp:11 kContainerVersion

_GEN = {hv.GenerationStrategy.kRandom: "random", hv.GenerationStrategy.kScaleRandom: "scale_random",
        hv.GenerationStrategy.kSandwich: "sandwich"}
_BIND = {hv.BindingStrategy.kIdLevel: "id_level", hv.BindingStrategy.kPermutation: "permutation",
         hv.BindingStrategy.kAppending: "appending"}
_METRIC = {hv.Metric.kHamming: "hamming", hv.Metric.kCosine: "cosine"}


def _json_double(x: float) -> str:
    """nlohmann::json's number_float dump: shortest round-trip digits, fixed
    notation for decimal exponents in (-4, 15], else d.ddde+XX (>= 2 digits)."""
    x = float(x)
    if x != x or x in (float("inf"), float("-inf")):
        return "null"
    if x == 0.0:
        return "-0.0" if str(x).startswith("-") else "0.0"
    sign = "-" if x < 0 else ""
    t = decimal.Decimal(repr(abs(x))).normalize().as_tuple()
    digits = "".join(map(str, t.digits))
    k, n = len(digits), len(digits) + t.exponent  # value = 0.digits * 10^n
    if k <= n <= 15:
        s = digits + "0" * (n - k) + ".0"
    elif 0 < n <= 15:
        s = digits[:n] + "." + digits[n:]
    elif -4 < n <= 0:
        s = "0." + "0" * (-n) + digits
    else:
        e = n - 1
        mant = digits if k == 1 else digits[0] + "." + digits[1:]
        s = f"{mant}e{'-' if e < 0 else '+'}{abs(e):02d}"
    return sign + s


def _dump(header: dict) -> bytes:
    parts = []
    for key in sorted(header):
        v = header[key]
        if isinstance(v, float):
            val = _json_double(v)
        elif isinstance(v, str):
            val = json.dumps(v)
        else:
            val = str(int(v))
        parts.append(f'"{key}":{val}')
    return ("{" + ",".join(parts) + "}").encode()


class _Reader:
    def __init__(self, data: bytes):
        self.b = memoryview(data)
        self.pos = 0

    def take(self, n: int) -> bytes:
        if self.pos + n > len(self.b):
            raise RuntimeError("unexpected end of stream")  # io.cpp read_bytes
        out = bytes(self.b[self.pos:self.pos + n])
        self.pos += n
        return out

    def u16(self) -> int:
        return struct.unpack("<H", self.take(2))[0]

    def u64(self) -> int:
        return struct.unpack("<Q", self.take(8))[0]

    def magic(self, m: str) -> None:
        if self.take(4) != m.encode():
            raise RuntimeError(f"bad magic, expected {m}")


# ------------------------------------------------------------------ HVPB ----
def write_packed(m: hv.PackedBitMatrix) -> bytes:
    """io.cpp:85-91."""
    words = np.ascontiguousarray(m.words, "<u4")
    return b"HVPB" + struct.pack("<HQQ", VERSION, m.rows, m.dim) + words.tobytes()


def _read_packed(r: _Reader) -> hv.PackedBitMatrix:
    """io.cpp:93-107."""
    r.magic("HVPB")
    version = r.u16()
    if version != VERSION:
        raise RuntimeError(f"unsupported packed-matrix version {version}")
    rows, dim = r.u64(), r.u64()
    W = hv.words_per_row(dim)
    words = np.frombuffer(r.take(rows * W * 4), "<u4").astype(np.uint32).reshape(rows, W)
    m = hv.PackedBitMatrix(rows, dim, words)
    if not m.padding_clean():
        raise RuntimeError("corrupt packed matrix: padding bits set")
    return m


def read_packed(data: bytes) -> hv.PackedBitMatrix:
    return _read_packed(_Reader(data))


def _header(r: _Reader, what: str) -> dict:
    n = r.u64()
    if r.pos + n > len(r.b):
        raise RuntimeError(f"truncated {what} header")
    text = r.take(n)
    try:
        return json.loads(text)
    except ValueError as e:
        raise RuntimeError(f"{what} header is not valid JSON: {e}") from None


# ------------------------------------------------------------------ HVCB ----
def save_codebook(c: hv.Codebook) -> bytes:
    """encoding.cpp:313-327."""
    text = _dump({"generation": _GEN[c.generation], "binding": _BIND[c.binding], "seed": c.seed,
                  "features": c.feature_count(), "bins": c.bin_count(), "dim": c.dim()})
    return (b"HVCB" + struct.pack("<HQ", VERSION, len(text)) + text + write_packed(c.id_vectors)
            + write_packed(c.value_vectors))


def load_codebook(data: bytes) -> hv.Codebook:
    """encoding.cpp:329-363."""
    r = _Reader(data)
    r.magic("HVCB")
    version = r.u16()
    if version != VERSION:
        raise RuntimeError(f"unsupported codebook version {version}")
    h = _header(r, "codebook")
    try:
        gen = {v: k for k, v in _GEN.items()}[h["generation"]]
        bind = {v: k for k, v in _BIND.items()}[h["binding"]]
        seed = int(h["seed"])
    except KeyError as e:
        raise RuntimeError(f"codebook header missing field: {e}") from None
    idv, val = _read_packed(r), _read_packed(r)
    if (idv.rows != h["features"] or val.rows != h["bins"] or idv.dim != h["dim"] or idv.dim != val.dim):
        raise RuntimeError("codebook header disagrees with stored matrices")
    return hv.Codebook(idv, val, gen, bind, seed)


# ------------------------------------------------------------------ HVMD ----
def save_model(m: hv.HDModel) -> bytes:
    """model.cpp:322-337."""
    cfg = m.config
    text = _dump({"class_count": cfg.class_count, "dim": cfg.dim, "gamma": float(cfg.gamma),
                  "metric": _METRIC[cfg.metric], "seed": cfg.seed})
    out = _io.BytesIO()
    out.write(b"HVMD" + struct.pack("<HQ", VERSION, len(text)) + text)
    out.write(write_packed(m.class_vectors))
    out.write(np.ascontiguousarray(m.accumulators, "<f8").tobytes())
    out.write(np.ascontiguousarray(m.class_weight, "<f8").tobytes())
    out.write(np.ascontiguousarray(m.sample_counts, "<u8").tobytes())
    return out.getvalue()


def load_model(data: bytes) -> hv.HDModel:
    """model.cpp:339-372 (tiebreak regenerated from the seed by make_empty_model)."""
    r = _Reader(data)
    r.magic("HVMD")
    version = r.u16()
    if version != VERSION:
        raise RuntimeError(f"unsupported model version {version}")
    n = r.u64()
    if r.pos + n > len(r.b):
        raise RuntimeError("truncated model header")
    try:
        h = json.loads(r.take(n))
        cfg = hv.ModelConfig(class_count=int(h["class_count"]), dim=int(h["dim"]), gamma=float(h["gamma"]),
                             metric={v: k for k, v in _METRIC.items()}[h["metric"]], seed=int(h["seed"]))
    except (ValueError, KeyError) as e:
        raise RuntimeError(f"bad model header: {e}") from None
    m = hv.make_empty_model(cfg)
    m.class_vectors = _read_packed(r)
    if m.class_vectors.rows != cfg.class_count or m.class_vectors.dim != cfg.dim:
        raise RuntimeError("model header disagrees with stored class vectors")
    C, D = cfg.class_count, cfg.dim
    m.accumulators = np.frombuffer(r.take(C * D * 8), "<f8").astype(np.float64).reshape(m.accumulators.shape)
    m.class_weight = np.frombuffer(r.take(C * 8), "<f8").astype(np.float64)
    m.sample_counts = np.frombuffer(r.take(C * 8), "<u8").astype(np.uint64)
    return m
