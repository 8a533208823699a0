"""The host-staged fold entry points (hv_fold_encode_train + hv_fold_predict,
the bench's e2e leg: host uint32 bins in, labels out) against the reference's
own run_fold_packed outputs at the UCI-HAR benchmark shape
(tests/golden/cases/bigpipe_har_d10k: F = 561, C = 6, D = 10000, 12,000 rows,
written by the reference library; experiment.cpp:148-178).

Both staging modes are covered — streamed (one persistent encoder launch per
row set waiting on the rows the copy stream has landed, hv_stage.cu
encode_host_bins_streamed) and the chunked pipeline (HVB200_STAGE_STREAM=0) —
at the default slot size and at 1 MB slots (many ramped chunks), plus the bad
bin path in the train and in the test rows (the reference's message, no hung
launch: the context runs a good fold right after).
"""
import ctypes as C
import os

import numpy as np
import pytest

import oracle_ref as O
from golden_io import Case

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(120)]

hv = pytest.importorskip("paper_2206_04746_b200.hypervec")
from paper_2206_04746_b200 import _native as N  # noqa: E402

MODES = [{}, {"HVB200_STAGE_MB": "1"}, {"HVB200_STAGE_STREAM": "0"},
         {"HVB200_STAGE_STREAM": "0", "HVB200_STAGE_MB": "1"}]


@pytest.fixture(scope="module")
def har():
    c = Case("bigpipe_har_d10k")
    rows, F, Cc, D, seed = c.int("rows"), c.int("features"), c.int("classes"), c.int("dim"), c.int("seed")
    ntr = c.int("train_rows")
    X, y = O.make_synth(rows, F, Cc, seed)
    disc = hv.fit_discretizer(X[:ntr], ntr, F, 16)
    bins = hv.discretize_matrix(X, rows, disc).reshape(rows, F).astype(np.uint32)
    np.testing.assert_array_equal(O.fnv_rows(bins), c["bins_fnv"])
    cb = hv.make_codebook(hv.GenerationStrategy.kRandom, hv.BindingStrategy.kIdLevel, F, 16, D,
                          hv.derive_seed(seed, 1))
    etb = hv.generate_random(1, D, hv.derive_seed(seed, 2))
    enc = hv.encode_batch(bins, rows, cb, etb).words[:ntr]
    return dict(c=c, rows=rows, F=F, C=Cc, D=D, ntr=ntr, y=np.ascontiguousarray(y[:ntr], np.int32),
                bins=np.ascontiguousarray(bins), idv=np.ascontiguousarray(cb.id_vectors.words),
                val=np.ascontiguousarray(cb.value_vectors.words), etb=np.ascontiguousarray(etb.words),
                mtb=np.ascontiguousarray(c["model_tiebreak"], np.uint32), enc=enc)


def _p(a):
    return C.c_void_p(a.ctypes.data)


def _fold(h, bins, env):
    """One fold through the C ABI; returns (labels, class rows, counts) or raises."""
    import torch

    old = {k: os.environ.get(k) for k in ("HVB200_STAGE_MB", "HVB200_STAGE_STREAM")}
    for k in old:
        os.environ.pop(k, None)
    os.environ.update(env)
    try:
        L = N.lib()
        ctx = N.context(0)
        ntr, nte, F = h["ntr"], h["rows"] - h["ntr"], h["F"]
        f = C.c_void_p()
        N.check(L.hv_fold_encode_train(ctx.handle, _p(bins), ntr, _p(h["y"]),
                                       C.c_void_p(bins.ctypes.data + ntr * F * 4), nte, F, _p(h["idv"]), _p(h["val"]),
                                       16, h["D"], _p(h["etb"]), h["C"], C.byref(f)))
        try:
            cp, rp = C.c_void_p(), C.c_void_p()
            N.check(L.hv_fold_counts(f, C.byref(cp), C.byref(rp)))
            W = (h["D"] + 31) // 32
            counts = np.empty(h["C"] * 32 * W, np.uint32)
            crow = np.empty(h["C"], np.uint64)
            torch.cuda.synchronize()
            _d2h(cp.value, counts)
            _d2h(rp.value, crow)
            labels = np.zeros(nte, np.int32)
            N.check(L.hv_fold_predict(ctx.handle, f, _p(h["mtb"]), _p(labels)))
        finally:
            L.hv_fold_destroy(f)
        return labels, crow, counts.reshape(h["C"], 32 * W)
    finally:
        for k, v in old.items():
            os.environ.pop(k, None)
            if v is not None:
                os.environ[k] = v


def _d2h(ptr, out):
    """Copies a library-owned device buffer into the host array `out`."""
    import torch

    class _CAI:  # zero-copy view of the device pointer
        __cuda_array_interface__ = {"shape": (out.nbytes,), "typestr": "|u1", "data": (ptr, False), "version": 3,
                                    "strides": None, "stream": None}

    out.view(np.uint8)[:] = torch.as_tensor(_CAI(), device="cuda:0").cpu().numpy()


def _recount(h):
    bits = np.unpackbits(h["enc"].view(np.uint8), axis=1, bitorder="little")[:, :h["D"]]
    W = (h["D"] + 31) // 32
    out = np.zeros((h["C"], 32 * W), np.uint32)
    for c in range(h["C"]):
        out[c, :h["D"]] = bits[h["y"] == c].sum(axis=0)
    return out


@pytest.mark.parametrize("env", MODES, ids=["streamed", "streamed-1MB", "chunked", "chunked-1MB"])
def test_fold_abi_matches_reference_pipeline(har, env):
    c = har["c"]
    labels, crow, counts = _fold(har, har["bins"], env)
    np.testing.assert_array_equal(crow, c["classical_counts"].astype(np.uint64))
    np.testing.assert_array_equal(counts[:, :har["D"]], _recount(har)[:, :har["D"]])
    np.testing.assert_array_equal(labels, c["classical_pred"])


@pytest.mark.parametrize("env", MODES[:3], ids=["streamed", "streamed-1MB", "chunked"])
@pytest.mark.parametrize("where", ["train", "test"])
def test_fold_abi_bad_bin_reports_and_recovers(har, env, where):
    bins = har["bins"].copy()
    r = 9000 if where == "train" else har["ntr"] + 1500
    assert (r < har["ntr"]) == (where == "train")
    bins[r, 5] = 16
    bins[r + 3, 0] = 99  # a later bad bin must not be the one reported
    with pytest.raises(Exception, match="feature 5 bin index 16 out of range \\(bins = 16\\)"):
        _fold(har, bins, env)
    labels, _, _ = _fold(har, har["bins"], env)  # the context is usable (no launch left waiting)
    np.testing.assert_array_equal(labels, har["c"]["classical_pred"])
