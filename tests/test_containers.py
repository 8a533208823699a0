"""HVPB / HVCB / HVMD containers (io.cpp:85-107, encoding.cpp:313-363,
model.cpp:322-372): the Python writers reproduce the reference's files byte
for byte (tests/golden/cases/containers, written by the reference library),
and the readers load them back. CPU only; the GPU test in test_gpu_eval.py
checks files written from GPU-trained models."""
import numpy as np
import pytest

from golden_io import Case

hv = pytest.importorskip("paper_2206_04746_b200.hypervec")
from paper_2206_04746_b200 import containers as io  # noqa: E402


def _b(c, key):
    return bytes(c[key].astype(np.uint8))


def test_packed_roundtrip_and_bytes():
    c = Case("containers")
    data = _b(c, "hvpb_encoded")
    m = io.read_packed(data)
    assert m.rows == 157 and m.dim == 1000
    assert io.write_packed(m) == data
    empty = _b(c, "hvpb_empty")
    e = io.read_packed(empty)
    assert e.rows == 0 and e.dim == 37 and io.write_packed(e) == empty
    p = Case("pipeline_odd")
    np.testing.assert_array_equal(m.words, p["encoded"])


def test_codebook_bytes_match_reference():
    c = Case("containers")
    cb = hv.make_codebook(0, 0, 13, 16, 1000, hv.derive_seed(12, 1))
    assert io.save_codebook(cb) == _b(c, "hvcb_random")
    cb2 = hv.make_codebook(hv.GenerationStrategy.kSandwich, hv.BindingStrategy.kPermutation, 5, 4, 64, 99)
    assert io.save_codebook(cb2) == _b(c, "hvcb_sandwich_perm")
    back = io.load_codebook(_b(c, "hvcb_sandwich_perm"))
    assert back.id_vectors == cb2.id_vectors and back.value_vectors == cb2.value_vectors
    assert (back.generation, back.binding, back.seed) == (cb2.generation, cb2.binding, 99)


def test_model_headers_and_bytes_match_reference():
    c = Case("containers")
    gammas = c["gammas"]
    for g, gamma in enumerate(gammas):
        cfg = hv.ModelConfig(class_count=2, dim=40, metric=g % 2, gamma=float(gamma), seed=1000 + g)
        want = _b(c, f"hvmd_gamma_{g}")
        assert io.save_model(hv.make_empty_model(cfg)) == want, gamma
        back = io.load_model(want)
        assert back.config.gamma == gamma and back.config.metric == g % 2 and back.config.seed == 1000 + g
    for key in ("hvmd_classical", "hvmd_online_b5"):
        data = _b(c, key)
        m = io.load_model(data)
        assert m.config.class_count == 3 and m.config.dim == 1000
        assert io.save_model(m) == data


def test_reader_errors_match_reference_messages():
    c = Case("containers")
    data = _b(c, "hvpb_encoded")
    with pytest.raises(RuntimeError, match="bad magic, expected HVPB"):
        io.read_packed(b"HVPC" + data[4:])
    with pytest.raises(RuntimeError, match="unsupported packed-matrix version 2"):
        io.read_packed(data[:4] + b"\x02\x00" + data[6:])
    with pytest.raises(RuntimeError, match="unexpected end of stream"):
        io.read_packed(data[:-1])
    bad = bytearray(data)
    bad[-1] |= 0x80  # dim 1000: the last word's top bits are padding
    with pytest.raises(RuntimeError, match="corrupt packed matrix: padding bits set"):
        io.read_packed(bytes(bad))
    with pytest.raises(RuntimeError, match="bad magic, expected HVMD"):
        io.load_model(data)
