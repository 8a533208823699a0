"""CPU checks of the C ABI boundary: the library loads, exports exactly what
include/hvb200.h declares, its host-side generators are bit-identical to the
reference (golden vectors), and compute entry points fail loudly without a
GPU (no CPU fallback)."""
import ctypes as C
import re

import numpy as np
import pytest
import torch

import oracle_ref as O
from golden_io import Case
from paper_2206_04746_b200 import _native as N

HAS_GPU = torch.cuda.is_available()


def declared_symbols():
    text = N.HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:[\w\s\*]+?)\b(hv_\w+)\s*\(", text, flags=re.M)))


def test_header_declares_all_bound_symbols():
    names = declared_symbols()
    assert len(names) >= 40
    assert set(names) == set(N.SIGNATURES), set(names) ^ set(N.SIGNATURES)


def test_library_exports_every_declared_symbol():
    L = N.lib()
    missing = [n for n in declared_symbols() if not hasattr(L, n)]
    assert not missing, missing
    assert L.hv_abi_version() == 1
    assert L.hv_words_per_row(10000) == 313
    assert L.hv_words_per_row(1) == 1 and L.hv_words_per_row(33) == 2


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(N.LIB_PATH)], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out, out


def test_rng_and_codebooks_match_reference_goldens():
    L = N.lib()
    c = Case("rng")
    ds = np.array([[L.hv_derive_seed(x, t) for t in range(1, 5)] for x in range(64)], np.uint64)
    np.testing.assert_array_equal(ds, c["derive_seed"])
    cb = Case("codebook")
    from paper_2206_04746_b200 import hypervec as hv
    np.testing.assert_array_equal(hv.generate_random(5, 10240, 99).words, cb["random_5x10240_s99"])
    np.testing.assert_array_equal(hv.generate_random(3, 33, 7).words, cb["random_3x33_s7"])
    np.testing.assert_array_equal(hv.generate_scale_random(16, 10240, 7).words, cb["scale_random_16x10240_s7"])
    np.testing.assert_array_equal(hv.generate_scale_random(17, 32, 1).words, cb["scale_random_17x32_s1"])
    np.testing.assert_array_equal(hv.generate_sandwich(8, 1000, 5).words, cb["sandwich_8x1000_s5"])
    np.testing.assert_array_equal(hv.generate_sandwich(5, 64, 3).words, cb["sandwich_5x64_s3"])
    for g, name in enumerate(("random", "scale_random", "sandwich")):
        book = hv.make_codebook(g, 0, 12, 8, 1024, 77)
        np.testing.assert_array_equal(book.id_vectors.words, cb[f"cb_{name}_id"])
        np.testing.assert_array_equal(book.value_vectors.words, cb[f"cb_{name}_value"])


def test_generator_errors_match_reference_messages():
    from paper_2206_04746_b200 import hypervec as hv
    with pytest.raises(hv.InvalidArgument, match=r"generate_scale_random: dim 31 too small for 17 bins"):
        hv.generate_scale_random(17, 31, 1)
    with pytest.raises(hv.InvalidArgument, match="generate_sandwich: dim must be even, got 999"):
        hv.generate_sandwich(4, 999, 5)
    with pytest.raises(hv.InvalidArgument, match="make_codebook: features and dim must be >= 1"):
        hv.make_codebook(0, 0, 0, 8, 64, 1)
    with pytest.raises(hv.InvalidArgument, match="make_codebook: need at least 2 bins"):
        hv.make_codebook(0, 0, 3, 1, 64, 1)


def test_make_empty_model_host_side():
    from paper_2206_04746_b200 import hypervec as hv
    m = hv.make_empty_model(hv.ModelConfig(class_count=3, dim=100, seed=5))
    tb = O.generate_random(1, 100, O.derive_seed(5, 3))
    np.testing.assert_array_equal(m.tiebreak.words, tb)
    for c in range(3):
        np.testing.assert_array_equal(m.class_vectors.words[c], tb[0])
    with pytest.raises(hv.InvalidArgument, match="need at least one class"):
        hv.make_empty_model(hv.ModelConfig(class_count=0, dim=100))
    with pytest.raises(hv.InvalidArgument, match="gamma must be >= 0"):
        hv.make_empty_model(hv.ModelConfig(class_count=2, dim=10, gamma=-0.5))


@pytest.mark.skipif(HAS_GPU, reason="checks the no-GPU behaviour")
def test_compute_fails_loudly_without_gpu():
    L = N.lib()
    h = C.c_void_p()
    st = L.hv_context_create(0, C.byref(h))
    assert st == N.HV_ERR_NO_DEVICE
    assert b"no CPU fallback" in L.hv_last_error()
    from paper_2206_04746_b200 import hypervec as hv
    N._contexts.clear()
    with pytest.raises(N.NoDevice):
        hv.encode_batch(np.zeros(4, np.uint32), 1, hv.make_codebook(0, 0, 4, 2, 64, 1), hv.generate_random(1, 64, 2))


def test_hamming_distance_words_host_helper():
    """The C ABI's host-only helper (the Python/drop-in API uses the device
    version hv_hamming_distance, tested on the GPU)."""
    import ctypes as C
    from paper_2206_04746_b200 import _native as N
    a = O.pack_rows(np.array([[1, 1, 0, 0, 1]], np.uint8))
    b = O.pack_rows(np.array([[1, 0, 0, 1, 1]], np.uint8))
    got = N.lib().hv_hamming_distance_words(a.ctypes.data_as(C.c_void_p), b.ctypes.data_as(C.c_void_p), 5)
    assert got == 2.0 / 5.0


def test_host_narrowing_matches_numpy_and_finds_first_bad_bin():
    """The host staging kernel of hv_encode_batch / hv_fold_* (csrc/hv_stage.cu),
    callable without a device: uint32 -> uint8 rows of pitch ldb, zero padding,
    and the first offending flat index (encoding.cpp:43-55 check order)."""
    import ctypes as C
    import numpy as np
    from paper_2206_04746_b200 import _native as N
    rng = np.random.default_rng(3)
    for rows, F, B, ldb in [(1, 1, 2, 64), (1000, 342, 16, 384), (777, 65, 7, 128), (0, 5, 4, 64)]:
        bins = rng.integers(0, B, (rows, F)).astype(np.uint32)
        out = np.full((max(rows, 1), ldb), 0xAB, np.uint8)
        bad = C.c_uint64()
        N.check(N.lib().hv_host_narrow_bins(bins.ctypes.data, rows, F, B, out.ctypes.data, ldb, C.byref(bad)))
        assert bad.value == 2**64 - 1
        if rows:
            np.testing.assert_array_equal(out[:rows, :F], bins.astype(np.uint8))
            assert not out[:rows, F:].any()
    # vector-path edges (AVX-512 streaming path needs 16-byte aligned rows; the
    # others take the AVX2 / scalar path): F a multiple of 16, ldb == F,
    # unaligned output, ldb not a multiple of 16, full 8-bit range
    for rows, F, B, ldb, off in [(300, 32, 16, 64, 0), (300, 48, 256, 48, 0), (200, 65, 16, 80, 1),
                                 (200, 65, 16, 70, 0), (50, 17, 256, 32, 0)]:
        bins = rng.integers(0, B, (rows, F)).astype(np.uint32)
        buf = np.full(rows * ldb + 64, 0xAB, np.uint8)
        base = (-buf.ctypes.data) % 64 + off
        out = buf[base:base + rows * ldb].reshape(rows, ldb)
        bad = C.c_uint64()
        N.check(N.lib().hv_host_narrow_bins(bins.ctypes.data, rows, F, B, out.ctypes.data, ldb, C.byref(bad)))
        assert bad.value == 2**64 - 1
        np.testing.assert_array_equal(out[:, :F], bins.astype(np.uint8))
        assert not out[:, F:].any()
    bins = rng.integers(0, 16, (100, 40)).astype(np.uint32)
    bins[77, 39] = 0x100  # truncates to 0 in uint8 but must still be reported
    out = np.zeros((100, 64), np.uint8)
    bad = C.c_uint64()
    N.check(N.lib().hv_host_narrow_bins(bins.ctypes.data, 100, 40, 16, out.ctypes.data, 64, C.byref(bad)))
    assert bad.value == 77 * 40 + 39
    bins = rng.integers(0, 16, (5000, 30)).astype(np.uint32)
    bins[4321, 7] = 16
    bins[4999, 0] = 99
    out = np.zeros((5000, 64), np.uint8)
    bad = C.c_uint64()
    N.check(N.lib().hv_host_narrow_bins(bins.ctypes.data, 5000, 30, 16, out.ctypes.data, 64, C.byref(bad)))
    assert bad.value == 4321 * 30 + 7
