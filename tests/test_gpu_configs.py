"""Parity at the BASELINE.json config shapes that round 1 left untested.

1. Reference-written pipelines at D = 10000 / 20000 / 1024 (tests/golden/cases/
   bigpipe_*, written by oracle/golden_gen.cpp linked against the reference
   library): UCI-HAR (F = 561, C = 6, 12,000 rows, online batches 256 / 1024 /
   8192), ISOLET (F = 617, C = 26, 2,500 rows), MNIST (F = 784, C = 10,
   D = 20000 and D = 1024). The whole run_fold_packed path (experiment.cpp:
   148-178) goes through the engine's C ABI: discretizer fit + discretize,
   encode, classical and online training, predict. Every encoded row and every
   fp64 accumulator row is compared through its FNV-1a digest, everything
   else in full — all bit-exact against the reference itself.
2. The C oracle at sizes the golden files cannot hold: UCI-HAR online with
   16,384+ rows at batch 256 / 1024 / 8192, Large online (C = 100, D = 32768,
   batch 1024, split-K tcgen05 scoring on), MNIST online at D = 1024 and
   20000 with batch 1024 (model.cpp:250-301, test_model.cpp:278-296).
"""
import numpy as np
import pytest
import torch

import oracle_ref as O
from golden_io import Case, cases

pytestmark = pytest.mark.gpu

hv = pytest.importorskip("paper_2206_04746_b200.hypervec")
dv = pytest.importorskip("paper_2206_04746_b200.device")
from paper_2206_04746_b200 import launch_count  # noqa: E402


def _u32(t):
    return t.cpu().numpy().view(np.uint32)


def _acc_fnv(acc2d):
    return O.fnv_rows(np.ascontiguousarray(acc2d, dtype=np.float64))


@pytest.mark.parametrize("name", cases("bigpipe_"))
def test_reference_pipeline_at_benchmark_shapes(name):
    c = Case(name)
    rows, F, C, D, seed = c.int("rows"), c.int("features"), c.int("classes"), c.int("dim"), c.int("seed")
    ntr = c.int("train_rows")
    gamma = c.float_bits("gamma_bits")
    X, y = O.make_synth(rows, F, C, seed)
    np.testing.assert_array_equal(O.fnv_rows(X), c["X_fnv"])
    np.testing.assert_array_equal(y, c["y"])
    before = launch_count()
    disc = hv.fit_discretizer(X[:ntr], ntr, F, 16)
    np.testing.assert_array_equal(disc.min, c["min"])
    np.testing.assert_array_equal(disc.max, c["max"])
    bins = hv.discretize_matrix(X, rows, disc).reshape(rows, F)
    np.testing.assert_array_equal(O.fnv_rows(bins.astype(np.uint32)), c["bins_fnv"])
    cb = hv.make_codebook(hv.GenerationStrategy.kRandom, hv.BindingStrategy.kIdLevel, F, 16, D,
                          hv.derive_seed(seed, 1))
    etb = hv.generate_random(1, D, hv.derive_seed(seed, 2))
    enc = hv.encode_batch(bins, rows, cb, etb)
    np.testing.assert_array_equal(O.fnv_rows(enc.words), c["encoded_fnv"])
    train = hv.PackedBitMatrix(ntr, D, enc.words[:ntr])
    test = hv.PackedBitMatrix(rows - ntr, D, enc.words[ntr:])
    cfg = hv.ModelConfig(class_count=C, dim=D, gamma=gamma, seed=seed)
    m = hv.train_classical(train, y[:ntr], cfg)
    np.testing.assert_array_equal(m.tiebreak.words, c["model_tiebreak"])
    np.testing.assert_array_equal(_acc_fnv(m.accumulators.reshape(C, D)), c["classical_acc_fnv"])
    np.testing.assert_array_equal(m.class_weight, c["classical_weight"])
    np.testing.assert_array_equal(m.sample_counts, c["classical_counts"])
    np.testing.assert_array_equal(m.class_vectors.words, c["classical_cv"])
    labels, dist = hv.predict_arrays(m, test)
    np.testing.assert_array_equal(labels, c["classical_pred"])
    np.testing.assert_array_equal(dist.view(np.uint64), c["classical_dist"].view(np.uint64))
    for b in c["batch_sizes"].tolist():
        k = f"online_b{b}"
        on = hv.train_online(train, y[:ntr], int(b), cfg)
        np.testing.assert_array_equal(_acc_fnv(on.accumulators.reshape(C, D)), c[k + "_acc_fnv"], err_msg=k)
        np.testing.assert_array_equal(on.class_weight.view(np.uint64), c[k + "_weight"].view(np.uint64))
        np.testing.assert_array_equal(on.sample_counts, c[k + "_counts"])
        np.testing.assert_array_equal(on.class_vectors.words, c[k + "_cv"])
        ol, _ = hv.predict_arrays(on, test)
        np.testing.assert_array_equal(ol, c[k + "_pred"])
    assert launch_count() > before


def _oracle_online(eng, cbk, enc, labels, bsz, C, D, gamma=1.0):
    acc, weight, counts, cv = eng.train_online(enc, labels, bsz, gamma)
    eng.dc.check()
    om = O.NaiveModel(C, D, _u32(cbk.model_tiebreak), O.HAMMING, gamma).train_online(
        _u32(enc), labels.cpu().numpy(), bsz)
    np.testing.assert_array_equal(acc.cpu().numpy().view(np.uint64), om.acc.view(np.uint64))
    np.testing.assert_array_equal(weight.cpu().numpy().view(np.uint64), om.weight.view(np.uint64))
    np.testing.assert_array_equal(counts.cpu().numpy().astype(np.uint64), om.counts.astype(np.uint64))
    np.testing.assert_array_equal(_u32(cv), om.class_vectors)
    return om


@pytest.mark.parametrize("bsz", [256, 1024, 8192])
def test_uci_har_online_batch_sweep_vs_oracle(bsz):
    """BASELINE configs[1]: UCI-HAR-shaped (F = 561, C = 6, D = 10000) online,
    18,000 rows (2+ batches even at 8192), bit-exact fp64 accumulators."""
    F, C, D, rows = 561, 6, 10000, 18000
    cbk = dv.DeviceCodebook.make(F, 16, D, seed=31)
    eng = dv.Engine(cbk, C)
    bins8, labels = eng.synth(0, rows, 0, 3)
    enc = eng.encode(bins8)
    om = _oracle_online(eng, cbk, enc, labels, bsz, C, D, gamma=0.9)
    # the trained model's predictions on fresh rows match the oracle's
    tb8, _ = eng.synth(rows, 2000, 0, 3)
    te = eng.encode(tb8)
    cvt = torch.from_numpy(O.pack_rows(om.cv).view(np.int32)).to(te.device)
    pred = eng.predict(cvt, te)
    ol, _ = om.predict(_u32(te))
    np.testing.assert_array_equal(pred.cpu().numpy(), ol)


def test_large_online_tensor_core_scoring_vs_oracle():
    """BASELINE configs[4] shape: C = 100, D = 32768, batch 1024, 5 batches
    after the bootstrap — the split-K tcgen05 scoring (default for many
    classes) against the oracle, not against the engine's own POPC path."""
    F, C, D, rows, bsz = 617, 100, 32768, 5 * 1024, 1024
    cbk = dv.DeviceCodebook.make(F, 16, D, seed=41)
    eng = dv.Engine(cbk, C)
    bins8, labels = eng.synth(0, rows, 0, 5)
    enc = eng.encode(bins8)
    _oracle_online(eng, cbk, enc, labels, bsz, C, D)


@pytest.mark.parametrize("D", [1024, 20000])
def test_mnist_online_batch_1024_vs_oracle(D):
    """BASELINE configs[2]: MNIST-shaped (F = 784, C = 10) online, batch 1024,
    at both ends of the D sweep."""
    F, C, rows = 784, 10, 8192
    cbk = dv.DeviceCodebook.make(F, 16, D, seed=51)
    eng = dv.Engine(cbk, C)
    bins8, labels = eng.synth(0, rows, 0, 6)
    enc = eng.encode(bins8)
    _oracle_online(eng, cbk, enc, labels, 1024, C, D, gamma=0.8)


def test_fast_encoder_ignores_row_padding_bytes():
    """bins8 bytes in [features, ldb) are padding the caller need not zero:
    the table encoder must give the same words as with zero padding (and as
    the generic encoder, which never reads them)."""
    F, C, D, rows = 342, 2, 10000, 3000
    cbk = dv.DeviceCodebook.make(F, 16, D, seed=61)
    eng = dv.Engine(cbk, C)
    bins8, _ = eng.synth(0, rows, 1, 4)
    want = eng.encode(bins8)
    noisy = bins8.clone()
    noisy[:, F:] = torch.randint(0, 256, (rows, noisy.shape[1] - F), dtype=torch.uint8, device=noisy.device)
    assert torch.equal(eng.encode(noisy), want)


def test_more_than_256_bins_rejected_loudly():
    """The device encoder stages one byte per bin: bin counts above 256 are
    refused with INVALID_ARGUMENT instead of corrupting neighbouring bytes."""
    F, D, B = 8, 256, 300
    cb = hv.make_codebook(hv.GenerationStrategy.kRandom, hv.BindingStrategy.kIdLevel, F, B, D, 5)
    tb = hv.generate_random(1, D, 6)
    bins = np.full((4, F), 299, np.uint32)
    with pytest.raises(hv.InvalidArgument, match="exceeds 256"):
        hv.encode_batch(bins, 4, cb, tb)


@pytest.mark.parametrize("D,C,rows", [(10000, 2, 9000), (10000, 3, 5000), (1024, 10, 7000), (32768, 5, 2500),
                                      (96, 4, 3000), (4000, 7, 4100), (20000, 31, 1500)])
def test_pitched_rows_counts_and_predict_match_unpitched(D, C, rows):
    """The engine's pitched HBM layout (rows padded to 16 bytes; TMA-staged
    class counts, uint4 predict) gives exactly the unpitched kernels' counts,
    labels, popcounts and distances — several row chunks, class segments that
    end inside a staged batch, two column ranges at D = 32768 — and garbage in
    the padding words is never read as data."""
    cbk = dv.DeviceCodebook.make(64, 16, D, seed=D + C)
    eng = dv.Engine(cbk, C)
    bins8, _ = eng.synth(0, rows, 0, 3)
    labels = torch.randint(0, C, (rows,), dtype=torch.int32, device="cuda")
    flat = eng.encode(bins8)
    pit = eng.pitched_empty(rows)
    pit.as_strided((rows, pit.stride(0)), (pit.stride(0), 1)).fill_(-1)  # poison the padding words
    eng.encode(bins8, out=pit)
    assert torch.equal(pit, flat)
    c1, r1 = eng.zero_counts()
    c2, r2 = eng.zero_counts()
    eng.class_counts(flat, labels, c1, r1)
    eng.class_counts(pit, labels, c2, r2)
    eng.dc.check()
    assert torch.equal(c1, c2) and torch.equal(r1, r2)
    cv = eng.binarize(c1, r1)
    n = rows
    d1 = torch.empty((n, C), dtype=torch.float64, device="cuda")
    d2 = torch.empty_like(d1)
    p1 = torch.empty((n, C), dtype=torch.int32, device="cuda")
    p2 = torch.empty_like(p1)
    l1 = eng.predict(cv, flat, distances=d1, popcounts=p1)
    l2 = eng.predict(cv, pit, distances=d2, popcounts=p2)
    eng.dc.check()
    assert torch.equal(l1, l2) and torch.equal(p1, p2) and torch.equal(d1.view(torch.int64), d2.view(torch.int64))
    # and against the oracle on a sample
    idx = np.arange(0, n, max(1, n // 50))
    m = O.NaiveModel(C, D, _u32(cbk.model_tiebreak))
    m.cv = O.unpack_rows(_u32(cv), D).copy()
    ol, od = m.predict(_u32(flat[torch.as_tensor(idx, device="cuda")]))
    np.testing.assert_array_equal(l2[torch.as_tensor(idx, device="cuda")].cpu().numpy(), ol)


def test_pitched_rows_rejected_for_many_classes():
    D, C = 4096, 40
    cbk = dv.DeviceCodebook.make(32, 16, D, seed=1)
    eng = dv.Engine(cbk, C)
    bins8, _ = eng.synth(0, 100, 0, 3)
    pit = eng.encode(bins8, pitched=True)
    if pit.stride(0) == pit.shape[1]:
        pytest.skip("W already a multiple of 4: pitched == unpitched")
    cv = torch.zeros((C, eng.W), dtype=torch.int32, device="cuda")
    with pytest.raises(Exception, match="fewer than 32 classes"):
        eng.predict(cv, pit)
    with pytest.raises(ValueError, match="unpitched"):
        eng.train_online(pit, torch.zeros(100, dtype=torch.int32, device="cuda"), 10)


@pytest.mark.parametrize("D", [10000, 1024, 333])
def test_two_class_label_scan_matches_full_scan_with_ties(D):
    """The two-class labels-only scan (2 popc(d & (q ^ c0)) > popc(d)) gives the
    same labels as the full two-distance scan, including exact ties (which keep
    class 0, the reference's strict <) and the extremes q = c0, q = c1."""
    C, rows = 2, 4000
    cbk = dv.DeviceCodebook.make(16, 16, D, seed=7)
    eng = dv.Engine(cbk, C)
    W = eng.W
    rng = np.random.default_rng(D)
    cvb = rng.integers(0, 2, (2, D), dtype=np.uint8)
    diff = np.nonzero(cvb[0] != cvb[1])[0]
    if diff.size % 2:
        cvb[1, diff[-1]] ^= 1
        diff = diff[:-1]
    q = np.repeat(cvb[:1], rows, axis=0)
    # exact ties: every third row takes class 1's value on half the differing bits
    for i in range(0, rows, 3):
        sel = rng.choice(diff, diff.size // 2, replace=False)
        q[i, sel] = cvb[1, sel]
    noise = rng.random((rows, D)) < 0.3
    q[1::3] ^= noise[1::3].astype(np.uint8)
    q[2] = cvb[1]
    qw = O.pack_rows(q)
    cvw = O.pack_rows(cvb)
    ldw = eng.pitched_empty(1).stride(0)
    store = torch.full((rows, ldw), -1, dtype=torch.int32, device="cuda")
    store[:, :W] = torch.from_numpy(qw.view(np.int32)).cuda()
    pit = store[:, :W]
    cv = torch.from_numpy(cvw.view(np.int32)).cuda()
    fast = eng.predict(cv, pit)
    pops = torch.empty((rows, 2), dtype=torch.int32, device="cuda")
    full = eng.predict(cv, pit, popcounts=pops)
    eng.dc.check()
    assert torch.equal(fast, full)
    p = pops.cpu().numpy()
    assert (p[::3, 0] == p[::3, 1]).all() and (fast[::3] == 0).all()
    assert fast[2].item() == 1


def test_single_pair_hamming_and_cosine_on_device():
    """model.cpp:169-196 single-pair helpers (drop-in overrides): device
    Hamming distance and sequential-fp64 cosine equal the oracle's, and zero
    vectors are domain errors like the reference."""
    rng = np.random.default_rng(5)
    for D in (1, 31, 333, 10000):
        a = O.pack_rows(rng.integers(0, 2, (1, D), dtype=np.uint8))[0]
        b = O.pack_rows(rng.integers(0, 2, (1, D), dtype=np.uint8))[0]
        want = float(np.unpackbits((a ^ b).view(np.uint8)).sum()) / D
        assert hv.hamming_distance_words(a, b, D) == want
        acc = rng.integers(-50, 50, D).astype(np.float64) * 0.37
        m = O.NaiveModel(1, D, O.generate_random(1, D, 3), O.COSINE)
        m.acc[:] = acc
        bits = O.unpack_rows(a.reshape(1, -1), D)[0]
        if bits.any():
            got = hv.cosine_similarity(acc, a, D)
            _, od = m.predict(a.reshape(1, -1))
            assert got == od[0, 0]
    with pytest.raises(hv.DomainError):
        hv.cosine_similarity(np.zeros(64), np.array([3, 0], np.uint32), 64)
    with pytest.raises(hv.DomainError):
        hv.cosine_similarity(np.ones(64), np.zeros(2, np.uint32), 64)
    with pytest.raises(hv.InvalidArgument, match="accumulator length != dim"):
        hv.cosine_similarity(np.ones(63), np.zeros(2, np.uint32), 64)


@pytest.mark.parametrize("D", [16, 48, 1024, 10000, 1000, 33, 1, 100, 36, 7])
def test_pack_unpack_vectorised_and_ballot_paths(D):
    """pack / unpack (kernels.cpp:44-73) on both device paths — 128-bit
    chunks when rows are a multiple of 16 bytes, warp ballots otherwise — are
    exact inverses matching the oracle, keep the padding bits zero, and report
    the first non-binary byte in row-major order like the reference."""
    rng = np.random.default_rng(D)
    rows = 3001
    dense = rng.integers(0, 2, (rows, D), dtype=np.uint8)
    p = hv.pack(hv.DenseBitMatrix(rows, D, dense))
    np.testing.assert_array_equal(p.words, O.pack_rows(dense))
    assert p.padding_clean()
    np.testing.assert_array_equal(hv.unpack(p).bits, dense)
    bad = dense.copy()
    flat = bad.reshape(-1)
    hits = sorted(rng.choice(flat.size, 3, replace=False))
    for k, h in enumerate(hits):
        flat[h] = 2 + k
    with pytest.raises(hv.InvalidArgument, match=rf"pack: non-binary entry {2} at flat index {hits[0]}"):
        hv.pack(hv.DenseBitMatrix(rows, D, bad))


@pytest.mark.parametrize("B,binding", [(32, 0), (17, 0), (32, 1), (24, 0)])
def test_table_encoder_up_to_32_bins_vs_generic_and_oracle(B, binding, monkeypatch):
    """17..32 bins take the table encoder's 32-bin tables (encoding.cpp:228-255
    accepts any bin count): equal to the generic kernel on 50,000 CHB-MIT-shaped
    rows with random bins, and to the oracle on a sample."""
    F, D, rows = 342, 10000, 50_000
    cbk = dv.DeviceCodebook.make(F, B, D, seed=77 + B, binding=binding)
    eng = dv.Engine(cbk, 2)
    bins = torch.randint(0, B, (rows, dv.bins_pitch(F)), dtype=torch.uint8, device="cuda")
    before = launch_count()
    fast = eng.encode(bins)
    assert launch_count() > before
    monkeypatch.setenv("HVB200_ENCODE_GENERIC", "1")
    generic = eng.encode(bins)
    torch.cuda.synchronize()
    assert torch.equal(fast, generic)
    idx = np.array([0, 1, rows // 2, rows - 1])
    b = bins[torch.as_tensor(idx, device="cuda")][:, :F].cpu().numpy().astype(np.uint32)
    want = O.encode_batch(b, _u32(cbk.id_vectors), _u32(cbk.value_vectors), B, D,
                          O.BIND_ID_LEVEL if binding == 0 else O.BIND_PERMUTATION, _u32(cbk.encode_tiebreak))
    np.testing.assert_array_equal(_u32(fast[torch.as_tensor(idx, device="cuda")]), want)


@pytest.mark.parametrize("extra", [1, 3])
def test_odd_row_pitch_takes_word_kernels_and_agrees(extra):
    """Rows whose pitch is not a multiple of 4 words (no 16-byte rows) take the
    word-wise count and scan kernels with the pitch honoured; results equal
    the unpitched ones. Empty inputs are no-ops."""
    D, C, rows = 10000, 3, 4100
    cbk = dv.DeviceCodebook.make(40, 16, D, seed=extra)
    eng = dv.Engine(cbk, C)
    bins8, _ = eng.synth(0, rows, 0, 5)
    labels = torch.randint(0, C, (rows,), dtype=torch.int32, device="cuda")
    flat = eng.encode(bins8)
    store = torch.full((rows, eng.W + extra), -1, dtype=torch.int32, device="cuda")
    odd = store[:, :eng.W]
    eng.encode(bins8, out=odd)
    assert torch.equal(odd, flat)
    c1, r1 = eng.zero_counts()
    c2, r2 = eng.zero_counts()
    eng.class_counts(flat, labels, c1, r1)
    eng.class_counts(odd, labels, c2, r2)
    assert torch.equal(c1, c2) and torch.equal(r1, r2)
    cv = eng.binarize(c1, r1)
    d1 = torch.empty((rows, C), dtype=torch.float64, device="cuda")
    d2 = torch.empty_like(d1)
    assert torch.equal(eng.predict(cv, flat, distances=d1), eng.predict(cv, odd, distances=d2))
    assert torch.equal(d1, d2)
    eng.class_counts(odd[:0], labels[:0], c2, r2)
    eng.predict(cv, odd[:0])
    eng.dc.check()
    assert torch.equal(c1, c2)
