"""GPU parity: the CUDA engine (through the C ABI) against the reference's
golden vectors and the C oracle. Bit-exact for every integer/bit result and
for the single-GPU online trainer's fp64 accumulators."""
import numpy as np
import pytest
import torch

import oracle_ref as O
from golden_io import Case, cases

pytestmark = pytest.mark.gpu

hv = pytest.importorskip("paper_2206_04746_b200.hypervec")
from paper_2206_04746_b200 import launch_count  # noqa: E402


def P(words, dim):
    return hv.PackedBitMatrix(words.shape[0], dim, words)


def Dn(bits):
    return hv.DenseBitMatrix(bits.shape[0], bits.shape[1], bits)


# ------------------------------------------------------------ kernels ----
@pytest.mark.parametrize("name", cases("kernels_"))
def test_bit_kernels_match_reference(name):
    c = Case(name)
    d = c.int("dim")
    a = c["a"]
    pa = hv.pack(Dn(a))
    np.testing.assert_array_equal(pa.words, c["pack_a"])
    assert pa.padding_clean()
    np.testing.assert_array_equal(hv.unpack(pa).bits, a)
    pb, pb1 = hv.pack(Dn(c["b"])), hv.pack(Dn(c["b1"]))
    np.testing.assert_array_equal(hv.xor_bind(pa, pb).words, c["xor_ab"])
    np.testing.assert_array_equal(hv.xor_bind(pa, pb1).words, c["xor_ab1"])
    for k, s in enumerate(c["shifts"]):
        np.testing.assert_array_equal(hv.rotate(pa, int(s)).words, c[f"rot_{k}"])
    np.testing.assert_array_equal(hv.horizontal_sum(pa), c["hsum"])
    t = hv.transpose(pa)
    assert t.rows == d and t.dim == a.shape[0] and t.padding_clean()
    np.testing.assert_array_equal(t.words, c["transpose"])
    np.testing.assert_array_equal(hv.vertical_sum(pa), c["vsum"])
    tb = hv.pack(Dn(c["maj_tiebreak"]))
    np.testing.assert_array_equal(hv.majority_binarize(c["maj_counts"], c.int("maj_n"), tb).words, c["maj_out"])


def test_kernel_properties_and_errors():
    rng = np.random.default_rng(0)
    d = Dn(rng.integers(0, 2, (37, 1000), dtype=np.uint8))
    p = hv.pack(d)
    assert hv.transpose(hv.transpose(p)) == p
    assert hv.rotate(hv.rotate(p, 47), 953) == p
    np.testing.assert_array_equal(hv.vertical_sum(p), hv.horizontal_sum(hv.transpose(p)))
    assert not np.any(hv.horizontal_sum(hv.xor_bind(p, p)))
    bad = d.bits.copy()
    bad[3, 7] = 2
    with pytest.raises(hv.InvalidArgument, match=r"pack: non-binary entry 2 at flat index 3007"):
        hv.pack(Dn(bad))
    with pytest.raises(hv.InvalidArgument, match=r"xor_bind: shape mismatch \(2x64 vs 3x64\)"):
        hv.xor_bind(hv.PackedBitMatrix(2, 64), hv.PackedBitMatrix(3, 64))
    with pytest.raises(hv.InvalidArgument, match="count 5 exceeds total 4 at position 0"):
        hv.majority_binarize(np.array([5], np.uint64), 4, hv.PackedBitMatrix(1, 1))
    with pytest.raises(hv.InvalidArgument, match="tiebreak must be 1x2"):
        hv.majority_binarize(np.array([1, 1], np.uint64), 4, hv.PackedBitMatrix(1, 3))
    # majority hand case (test_kernels.cpp:176-188)
    tb = np.zeros((1, 6), np.uint8)
    tb[0, 2] = 1
    got = hv.majority_binarize(np.array([3, 1, 2, 2, 4, 0], np.uint64), 4, hv.pack(Dn(tb)))
    np.testing.assert_array_equal(hv.unpack(got).bits[0], [1, 0, 1, 0, 1, 0])
    # empty shapes
    assert hv.vertical_sum(hv.PackedBitMatrix(0, 70)).tolist() == [0] * 70
    assert hv.horizontal_sum(hv.PackedBitMatrix(0, 70)).size == 0


def test_launch_counter():
    before = launch_count()
    hv.pack(Dn(np.ones((2, 40), np.uint8)))
    assert launch_count() > before


# -------------------------------------------------------- discretizer ----
def test_discretizer_matches_reference():
    c = Case("discretize")
    data = c["data"]
    d = hv.fit_discretizer(data, data.shape[0], data.shape[1], 16)
    np.testing.assert_array_equal(d.min, c["min"])
    np.testing.assert_array_equal(d.max, c["max"])
    np.testing.assert_array_equal(hv.discretize_matrix(data, data.shape[0], d).reshape(data.shape), c["bins"])
    pr = c["probe"]
    np.testing.assert_array_equal(hv.discretize_matrix(pr, pr.shape[0], d).reshape(pr.shape), c["probe_bins"])
    # known answers (test_encoding.cpp:60-82)
    q = hv.Discretizer(np.array([0.0]), np.array([1.0]), 4)
    got = [int(hv.discretize([x], q)[0]) for x in (0.0, 0.24, 0.25, 0.74, 0.75, 1.0, -5.0, 42.0, float("nan"))]
    assert got == [0, 0, 1, 2, 3, 3, 0, 3, 0]
    with pytest.raises(hv.InvalidArgument, match="empty training matrix"):
        hv.fit_discretizer(np.zeros(0), 0, 2, 4)
    with pytest.raises(hv.InvalidArgument, match="need at least 2 bins"):
        hv.fit_discretizer(np.zeros(6), 3, 2, 1)


def test_fit_discretizer_nan_first_row_and_many_blocks():
    rng = np.random.default_rng(1)
    data = rng.normal(size=(20000, 5))
    data[0, 1] = np.nan
    data[777, 2] = np.nan
    d = hv.fit_discretizer(data, 20000, 5, 16)
    mn, mx = O.fit_discretizer(data, 16)
    np.testing.assert_array_equal(d.min, mn)
    np.testing.assert_array_equal(d.max, mx)


# ------------------------------------------------------------- encode ----
def _codebook(c):
    return hv.make_codebook(c.int("generation"), c.int("binding"), c.int("F"), c.int("B"), c.int("D"), c.int("seed"))


@pytest.mark.parametrize("name", cases("encode_"))
def test_encode_matches_reference(name):
    c = Case(name)
    cb = _codebook(c)
    tb = hv.generate_random(1, c.int("D"), c.int("tiebreak_seed"))
    got = hv.encode_batch(c["bins"], c.int("rows"), cb, tb)
    assert got.padding_clean()
    np.testing.assert_array_equal(got.words, c["out"])


def test_encode_errors_match_reference_messages():
    cb = hv.make_codebook(0, 0, 2, 4, 64, 17)
    tb = hv.generate_random(1, 64, 18)
    with pytest.raises(hv.InvalidArgument, match=r"encode: feature 1 bin index 4 out of range \(bins = 4\)"):
        hv.encode(np.array([0, 4]), cb, tb)
    with pytest.raises(hv.InvalidArgument, match="encode: expected 2 bin indices, got 1"):
        hv.encode(np.array([0]), cb, tb)
    with pytest.raises(hv.InvalidArgument, match="tiebreak must be 1 x dim"):
        hv.encode(np.array([0, 1]), cb, hv.generate_random(1, 63, 18))
    app = hv.make_codebook(0, 2, 40, 2, 32, 15)
    with pytest.raises(hv.InvalidArgument, match="encode: appending needs dim >= feature count"):
        hv.encode(np.zeros(40, np.uint32), app, hv.generate_random(1, 32, 16))
    # a bad bin in a later row is found on the device and reported with its feature
    big = np.zeros((5000, 2), np.uint32)
    big[4321, 0] = 9
    with pytest.raises(hv.InvalidArgument, match=r"feature 0 bin index 9 out of range"):
        hv.encode_batch(big, 5000, cb, tb)


@pytest.mark.parametrize("F,B,D,rows", [(617, 16, 10000, 300), (342, 16, 10000, 300), (784, 16, 1024, 200),
                                        (784, 16, 20000, 64), (561, 16, 10000, 100), (100, 16, 32768, 40),
                                        (5, 16, 33, 700), (1, 16, 31, 50), (16, 2, 32, 100), (2000, 16, 512, 40),
                                        (33, 32, 777, 100)])
def test_encode_random_vs_oracle(F, B, D, rows):
    rng = np.random.default_rng(F * 7 + D)
    bins = rng.integers(0, B, (rows, F)).astype(np.uint32)
    cb = hv.make_codebook(0, 0, F, B, D, 1000 + F)
    tb = hv.generate_random(1, D, 2000 + D)
    got = hv.encode_batch(bins, rows, cb, tb)
    want = O.encode_batch(bins, cb.id_vectors.words, cb.value_vectors.words, B, D, O.BIND_ID_LEVEL, tb.words)
    np.testing.assert_array_equal(got.words, want)


@pytest.mark.parametrize("env", [{"HVB200_TT_SHAPE": "4,8,1"}, {"HVB200_TT_SHAPE": "3,8,1"},
                                 {"HVB200_TT_SHAPE": "2,8,1"}, {"HVB200_TT_SHAPE": "1,8,2"},
                                 {"HVB200_TT_BLOCK_ROWS": "64"}])
@pytest.mark.parametrize("F,D", [(342, 10000), (617, 1000), (40, 333), (130, 64)])
def test_encode_fast_variants_vs_oracle(env, F, D, monkeypatch):
    """Every instantiated shape of the table-lookup encoder against the oracle: tail chunks of 16/32/48 features, F < 64,
    partial word slices, partial row tiles and (small blocks) table rebuilds."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    B, rows = 16, 700
    rng = np.random.default_rng(F + D)
    bins = rng.integers(0, B, (rows, F)).astype(np.uint32)
    cb = hv.make_codebook(0, 0, F, B, D, 77 + F)
    tb = hv.generate_random(1, D, 78 + D)
    got = hv.encode_batch(bins, rows, cb, tb)
    want = O.encode_batch(bins, cb.id_vectors.words, cb.value_vectors.words, B, D, O.BIND_ID_LEVEL, tb.words)
    np.testing.assert_array_equal(got.words, want)


@pytest.mark.parametrize("binding", [1, 2])
@pytest.mark.parametrize("D", [33, 1000, 10240])
def test_permutation_and_appending_vs_oracle(binding, D):
    rng = np.random.default_rng(D + binding)
    F = 24 if binding == 1 else 17
    bins = rng.integers(0, 7, (30, F)).astype(np.uint32)
    cb = hv.make_codebook(1 if D >= 32 else 0, binding, F, 7, D, 5)
    tb = hv.generate_random(1, D, 6)
    got = hv.encode_batch(bins, 30, cb, tb)
    want = O.encode_batch(bins, cb.id_vectors.words, cb.value_vectors.words, 7, D, binding, tb.words)
    np.testing.assert_array_equal(got.words, want)


@pytest.mark.parametrize("binding", [0, 1])
def test_encode_fast_and_generic_kernels_agree_at_scale(binding):
    """Size-independent property at bench scale: both device encoders give
    identical words for 200k CHB-MIT-shaped rows, for ID-level and for
    permutation binding (the table encoder with rotated level vectors); a
    sample is oracle-checked."""
    from paper_2206_04746_b200 import device as dv
    import os
    F, B, D, C, rows = 342, 16, 10000, 2, 200_000
    cbk = dv.DeviceCodebook.make(F, B, D, seed=3, binding=binding)
    eng = dv.Engine(cbk, C)
    bins8, labels = eng.synth(0, rows, 1, 7)
    fast = eng.encode(bins8)
    os.environ["HVB200_ENCODE_GENERIC"] = "1"
    try:
        slow = eng.encode(bins8)
    finally:
        del os.environ["HVB200_ENCODE_GENERIC"]
    torch.cuda.synchronize()
    assert torch.equal(fast, slow)
    idx = np.array([0, 1, 119, 120, 65535, 131071, rows - 1])
    b = bins8[idx][:, :F].cpu().numpy().astype(np.uint32)
    ref_b, _ = O.synth_c(0, rows, F, C, B, 1, 7)
    np.testing.assert_array_equal(b, ref_b[idx])
    want = O.encode_batch(b, cbk.id_vectors.cpu().numpy().view(np.uint32), cbk.value_vectors.cpu().numpy().view(np.uint32),
                          B, D, binding, cbk.encode_tiebreak.cpu().numpy().view(np.uint32))
    np.testing.assert_array_equal(fast[idx].cpu().numpy().view(np.uint32), want)


# ---------------------------------------------------------- pipelines ----
def _split(c):
    enc = c["encoded"]
    ntr = c.int("train_rows")
    return enc[:ntr], enc[ntr:], c["y"], ntr


@pytest.mark.parametrize("name", cases("pipeline_"))
def test_pipeline_matches_reference(name):
    c = Case(name)
    n, F, C, D, seed = c.int("rows"), c.int("features"), c.int("classes"), c.int("dim"), c.int("seed")
    gamma = c.float_bits("gamma_bits")
    ntr = c.int("train_rows")
    d = hv.fit_discretizer(c["X"][:ntr], ntr, F, 16)
    bins = hv.discretize_matrix(c["X"], n, d)
    np.testing.assert_array_equal(bins.reshape(n, F), c["bins"])
    cb = hv.make_codebook(0, 0, F, 16, D, hv.derive_seed(seed, 1))
    etb = hv.generate_random(1, D, hv.derive_seed(seed, 2))
    enc = hv.encode_batch(bins, n, cb, etb)
    np.testing.assert_array_equal(enc.words, c["encoded"])
    train = P(enc.words[:ntr], D)
    test = P(enc.words[ntr:], D)
    y = c["y"]
    cfg = hv.ModelConfig(class_count=C, dim=D, gamma=gamma, seed=seed)
    m = hv.train_classical(train, y[:ntr], cfg)
    np.testing.assert_array_equal(m.accumulators.reshape(C, D), c["classical_acc"])
    np.testing.assert_array_equal(m.class_weight, c["classical_weight"])
    np.testing.assert_array_equal(m.sample_counts, c["classical_counts"])
    np.testing.assert_array_equal(m.class_vectors.words, c["classical_cv"])
    np.testing.assert_array_equal(m.tiebreak.words, c["model_tiebreak"])
    labels, dist = hv.predict_arrays(m, test)
    np.testing.assert_array_equal(labels, c["classical_pred"])
    np.testing.assert_array_equal(dist, c["classical_dist"])
    for bsz in c["batch_sizes"]:
        k = f"online_b{int(bsz)}"
        on = hv.train_online(train, y[:ntr], int(bsz), cfg)
        # bit-exact fp64: same per-element sequence of IEEE additions
        np.testing.assert_array_equal(on.accumulators.reshape(C, D), c[k + "_acc"])
        np.testing.assert_array_equal(on.class_weight, c[k + "_weight"])
        np.testing.assert_array_equal(on.sample_counts, c[k + "_counts"])
        np.testing.assert_array_equal(on.class_vectors.words, c[k + "_cv"])
        np.testing.assert_array_equal(hv.predict_arrays(on, test)[0], c[k + "_pred"])
    ccfg = hv.ModelConfig(class_count=C, dim=D, metric=hv.Metric.kCosine, gamma=gamma, seed=seed)
    cm = hv.train_classical(train, y[:ntr], ccfg)
    cl, cd = hv.predict_arrays(cm, test)
    np.testing.assert_array_equal(cl, c["cosine_pred"])
    np.testing.assert_array_equal(cd, c["cosine_dist"])  # sequential fp64 like the reference
    con = hv.train_online(train, y[:ntr], int(c["batch_sizes"][0]), ccfg)
    np.testing.assert_array_equal(con.accumulators.reshape(C, D), c["cosine_online_acc"])
    np.testing.assert_array_equal(con.class_weight, c["cosine_online_weight"])
    np.testing.assert_array_equal(con.class_vectors.words, c["cosine_online_cv"])


def test_online_update_single_batch_matches_reference():
    c = Case("online_update")
    C_, D = c.int("classes"), c.int("dim")
    cfg = hv.ModelConfig(class_count=C_, dim=D, gamma=c.float_bits("gamma_bits"), seed=c.int("seed"))
    m = hv.train_classical(hv.pack(Dn(c["base"])), c["base_y"], cfg)
    hv.online_update(m, hv.pack(Dn(c["batch"])), c["y"], hv.freeze(m))
    np.testing.assert_array_equal(m.accumulators.reshape(C_, D), c["acc"])
    np.testing.assert_array_equal(m.class_weight, c["weight"])
    np.testing.assert_array_equal(m.sample_counts, c["counts"])
    np.testing.assert_array_equal(m.class_vectors.words, c["cv"])


def test_model_known_answers_and_errors():
    x = hv.pack(Dn(np.array([[1, 1, 0], [1, 0, 0], [0, 1, 1]], np.uint8)))
    cfg = hv.ModelConfig(class_count=2, seed=6)
    m = hv.train_classical(x, [0, 0, 1], cfg)
    assert m.accumulator_row(0).tolist() == [2.0, 1.0, 0.0]
    assert m.class_weight[0] == 2.0 and m.sample_counts.tolist() == [2, 1]
    assert m.class_vectors.bit(0, 0) and not m.class_vectors.bit(0, 2)
    assert m.class_vectors.bit(0, 1) == m.tiebreak.bit(0, 1)
    with pytest.raises(hv.InvalidArgument, match=r"train_classical: label 2 at row 2 out of range \(classes = 2\)"):
        hv.train_classical(x, [0, 0, 2], cfg)
    with pytest.raises(hv.InvalidArgument, match="train_classical: 2 labels for 3 rows"):
        hv.train_classical(x, [0, 0], cfg)
    with pytest.raises(hv.InvalidArgument, match="train_online: batch_size must be >= 1"):
        hv.train_online(x, [0, 0, 1], 0, cfg)
    with pytest.raises(hv.InvalidArgument, match="predict: query dim != model dim"):
        hv.predict(m, hv.PackedBitMatrix(1, 5))
    # delta = 0 exact no-op; gamma = 0 exact (acceptance.cpp:255-291)
    xs = hv.pack(Dn(np.array([[1, 0, 1, 1], [0, 1, 0, 0]], np.uint8)))
    m = hv.train_classical(xs, [0, 1], hv.ModelConfig(class_count=2, seed=8))
    before = m.accumulators.copy()
    hv.online_update(m, hv.pack(Dn(np.array([[1, 0, 1, 1]], np.uint8))), [0], hv.freeze(m))
    assert np.array_equal(m.accumulators, before) and m.sample_counts[0] == 2
    m = hv.train_classical(xs, [0, 1], hv.ModelConfig(class_count=2, gamma=0.0, seed=9))
    before = m.accumulators.copy()
    hv.online_update(m, hv.pack(Dn(np.array([[1, 0, 1, 1]], np.uint8))), [1], hv.freeze(m))
    assert np.array_equal(m.accumulators[:4], before[:4]) and m.accumulators[4] > before[4]
    # predict known answers and lowest-index ties (test_model.cpp:298-320)
    xx = hv.pack(Dn(np.array([[1, 1, 1, 1], [0, 0, 0, 0], [1, 1, 0, 0]], np.uint8)))
    m = hv.train_classical(xx, [0, 1, 2], hv.ModelConfig(class_count=3, seed=12))
    p = hv.predict(m, xx)
    assert [q.label for q in p] == [0, 1, 2] and p[0].distances.tolist()[:2] == [0.0, 1.0]
    tie = hv.predict(m, hv.pack(Dn(np.array([[1, 1, 0, 1]], np.uint8))))
    assert tie[0].distances[0] == tie[0].distances[2] and tie[0].label == 0
    # cosine: empty class never selected, zero query is a domain error
    cm = hv.train_classical(hv.pack(Dn(np.array([[1, 1, 0, 0], [0, 0, 1, 1]], np.uint8))), [0, 1],
                            hv.ModelConfig(class_count=3, metric=hv.Metric.kCosine, seed=14))
    cp = hv.predict(cm, hv.pack(Dn(np.array([[1, 0, 0, 0], [0, 0, 0, 1]], np.uint8))))
    assert [q.label for q in cp] == [0, 1] and cp[0].distances[2] == -np.inf
    with pytest.raises(hv.DomainError):
        hv.predict(cm, hv.PackedBitMatrix(1, 4))


@pytest.mark.parametrize("bsz", [1, 7, 64, 1000])
def test_online_random_vs_oracle_bitexact(bsz):
    rng = np.random.default_rng(bsz)
    C, D, n = 5, 1000, 700
    centers = rng.integers(0, 2, (C, D), dtype=np.uint8)
    y = rng.integers(0, C, n).astype(np.int32)
    enc = O.pack_rows(centers[y] ^ (rng.random((n, D)) < 0.3).astype(np.uint8))
    cfg = hv.ModelConfig(class_count=C, dim=D, gamma=0.7, seed=21)
    on = hv.train_online(P(enc, D), y, bsz, cfg)
    oo = O.NaiveModel(C, D, on.tiebreak.words, O.HAMMING, 0.7).train_online(enc, y, bsz)
    np.testing.assert_array_equal(on.accumulators.reshape(C, D), oo.acc)
    np.testing.assert_array_equal(on.class_weight, oo.weight)
    np.testing.assert_array_equal(on.class_vectors.words, oo.class_vectors)


@pytest.mark.parametrize("C,D,n,bsz", [(2, 1000, 900, 300), (1, 333, 600, 64), (3, 1000, 700, 256), (8, 333, 600, 64),
                                       (26, 2048, 800, 100), (32, 777, 500, 128), (100, 4096, 600, 512),
                                       (40, 64, 300, 1), (3, 70, 257, 256), (6, 10000, 2100, 1024), (6, 2000, 300, 32),
                                       (100, 1500, 400, 7), (64, 10000, 700, 256), (130, 3000, 500, 128),
                                       (100, 4096, 600, 100), (2, 5000, 900, 300), (2, 10240, 700, 256),
                                       (2, 10272, 600, 128)])
def test_online_modes_vs_oracle_bitexact(C, D, n, bsz):
    """Every path of the persistent online trainer against the oracle:
    MERGED (C <= 2), LISTS with warp-per-row scoring (2 < C < 32) and with
    lane-per-class scoring (C >= 32); partial chunks, one-row batches, tails."""
    rng = np.random.default_rng(C * 1000 + bsz)
    centers = rng.integers(0, 2, (C, D), dtype=np.uint8)
    y = rng.integers(0, C, n).astype(np.int32)
    enc = O.pack_rows(centers[y] ^ (rng.random((n, D)) < 0.35).astype(np.uint8))
    cfg = hv.ModelConfig(class_count=C, dim=D, gamma=0.9, seed=C + D)
    on = hv.train_online(P(enc, D), y, bsz, cfg)
    oo = O.NaiveModel(C, D, on.tiebreak.words, O.HAMMING, 0.9).train_online(enc, y, bsz)
    np.testing.assert_array_equal(on.accumulators.reshape(C, D), oo.acc)
    np.testing.assert_array_equal(on.class_weight, oo.weight)
    np.testing.assert_array_equal(on.sample_counts, oo.counts)
    np.testing.assert_array_equal(on.class_vectors.words, oo.class_vectors)


@pytest.mark.parametrize("bsz,p1,dyn", [(1024, 0.01, "1"), (2048, 0.3, "1"), (1024, 0.01, "0"), (256, 0.01, "1")])
def test_online_two_class_dynamic_items_vs_oracle_bitexact(bsz, p1, dyn, monkeypatch):
    """Two classes at D = 10,000: 158 narrow replay items on at most one CTA
    per SM, the items past the item CTAs drawn dynamically (batches >= 1,024
    rows), and class-weight tasks that skip groups without true samples — an
    unbalanced (CHB-MIT-like) and a balanced label mix, against the oracle."""
    monkeypatch.setenv("HVB200_ONLINE_DYNAMIC", dyn)
    rng = np.random.default_rng(int(p1 * 1000) + bsz)
    C, D, n = 2, 10000, 5000
    centers = rng.integers(0, 2, (C, D), dtype=np.uint8)
    y = (rng.random(n) < p1).astype(np.int32)
    enc = O.pack_rows(centers[y] ^ (rng.random((n, D)) < 0.4).astype(np.uint8))
    cfg = hv.ModelConfig(class_count=C, dim=D, gamma=0.6, seed=77)
    on = hv.train_online(P(enc, D), y, bsz, cfg)
    oo = O.NaiveModel(C, D, on.tiebreak.words, O.HAMMING, 0.6).train_online(enc, y, bsz)
    np.testing.assert_array_equal(on.accumulators.reshape(C, D), oo.acc)
    np.testing.assert_array_equal(on.class_weight, oo.weight)
    np.testing.assert_array_equal(on.sample_counts, oo.counts)
    np.testing.assert_array_equal(on.class_vectors.words, oo.class_vectors)


@pytest.mark.parametrize("C,D,n,bsz", [(1, 100, 50, 1), (2, 10000, 300, 1), (6, 10000, 400, 5), (6, 1000, 257, 16),
                                        (26, 2048, 200, 7), (32, 333, 130, 64), (3, 31, 90, 4), (13, 8192, 100, 33),
                                        (6, 20000, 120, 2)])
def test_online_cluster_path_vs_oracle_bitexact(C, D, n, bsz, monkeypatch):
    """The small-batch cluster trainer (one 8-CTA cluster, word slices resident
    in shared memory, DSMEM popcount reduction), forced for batches up to 64
    rows: accumulators, weights, counts and class vectors bit-exact vs the
    oracle — including slices narrower than a CTA's threads and D % 32 != 0.
    Shapes whose slices do not fit shared memory fall back to the persistent
    kernel and must agree just the same."""
    monkeypatch.setenv("HVB200_ONLINE_CLUSTER", "64")
    rng = np.random.default_rng(C * 77 + bsz + D)
    centers = rng.integers(0, 2, (C, D), dtype=np.uint8)
    y = rng.integers(0, C, n).astype(np.int32)
    enc = O.pack_rows(centers[y] ^ (rng.random((n, D)) < 0.3).astype(np.uint8))
    cfg = hv.ModelConfig(class_count=C, dim=D, gamma=0.7, seed=C + D + 1)
    before = launch_count()
    on = hv.train_online(P(enc, D), y, bsz, cfg)
    assert launch_count() > before
    oo = O.NaiveModel(C, D, on.tiebreak.words, O.HAMMING, 0.7).train_online(enc, y, bsz)
    np.testing.assert_array_equal(on.accumulators.reshape(C, D), oo.acc)
    np.testing.assert_array_equal(on.class_weight, oo.weight)
    np.testing.assert_array_equal(on.sample_counts, oo.counts)
    np.testing.assert_array_equal(on.class_vectors.words, oo.class_vectors)


@pytest.mark.parametrize("popc", ["0", "1", "imma"])
@pytest.mark.parametrize("C,D,n", [(32, 1000, 257), (33, 64, 100), (100, 4096, 300), (64, 10000, 70), (40, 31, 33),
                                   (129, 500, 40), (200, 96, 77), (64, 33, 300), (100, 1000, 129)])
def test_predict_many_classes_tiled_vs_oracle(C, D, n, popc, monkeypatch):
    """The many-class Hamming scans (C >= 32) — tcgen05 tensor cores (default
    from 64 classes), legacy mma.sync (HVB200_PREDICT_IMMA) and the CTA-tiled
    POPC scan (HVB200_PREDICT_POPC): labels and fp64 distances
    bit-exact vs the oracle, including ties between classes (duplicated class
    vectors must resolve to the lowest class) and several class tiles."""
    if popc == "1":
        monkeypatch.setenv("HVB200_PREDICT_POPC", "1")
    if popc == "imma":
        monkeypatch.setenv("HVB200_PREDICT_IMMA", "1")
    rng = np.random.default_rng(C + D + n)
    W = (D + 31) // 32
    cvb = rng.integers(0, 2, (C, D), dtype=np.uint8)
    cvb[C // 2] = cvb[1]  # a duplicate class: ties must pick class 1
    y = rng.integers(0, C, n).astype(np.int32)
    enc = O.pack_rows(cvb[y] ^ (rng.random((n, D)) < 0.3).astype(np.uint8))
    m = O.NaiveModel(C, D, O.generate_random(1, D, 3)).train_classical(enc, y)
    model = hv.make_empty_model(hv.ModelConfig(class_count=C, dim=D, seed=3))
    model.class_vectors.words[:] = O.pack_rows(cvb)
    m.cv[:] = cvb
    labels, dist = hv.predict_arrays(model, P(enc, D))
    ol, od = m.predict(enc)
    np.testing.assert_array_equal(labels, ol)
    np.testing.assert_array_equal(dist, od)


# --------------------------------------------------- device pipeline ----
def test_device_classical_and_predict_vs_oracle():
    from paper_2206_04746_b200 import device as dv
    F, B, D, C, rows = 617, 16, 10000, 26, 3000
    cbk = dv.DeviceCodebook.make(F, B, D, seed=9)
    eng = dv.Engine(cbk, C)
    bins8, labels = eng.synth(0, rows, 0, 7)
    enc = eng.encode(bins8)
    cv, counts, crow = eng.train_classical(enc[:2400], labels[:2400])
    pred = eng.predict(cv, enc[2400:])
    eng.dc.check()
    encn = enc.cpu().numpy().view(np.uint32)
    yn = labels.cpu().numpy()
    om = O.NaiveModel(C, D, cbk.model_tiebreak.cpu().numpy().view(np.uint32)).train_classical(encn[:2400], yn[:2400])
    np.testing.assert_array_equal(counts[:, :D].cpu().numpy().astype(np.float64), om.acc)
    np.testing.assert_array_equal(crow.cpu().numpy(), om.counts.astype(np.int64))
    np.testing.assert_array_equal(cv.cpu().numpy().view(np.uint32), om.class_vectors)
    ol, _ = om.predict(encn[2400:])
    np.testing.assert_array_equal(pred.cpu().numpy(), ol)


@pytest.mark.parametrize("D", [10000, 4096, 1000])
@pytest.mark.parametrize("skip", [0, 1, 3])
def test_device_predict_many_classes_offset_rows(D, skip):
    """Device many-class scan on a row view starting `skip` rows in: the
    tcgen05 path for 16-byte-aligned row data (aligned rows, or the 48-byte
    window copies when W % 4 != 0), the mma.sync path otherwise — labels and
    popcounts bit-exact vs the oracle."""
    from paper_2206_04746_b200 import device as dv
    C, rows = 70, 600
    cbk = dv.DeviceCodebook.make(64, 16, D, seed=5)
    eng = dv.Engine(cbk, C)
    bins8, labels = eng.synth(0, rows, 0, 11)
    enc = eng.encode(bins8)
    cv, _, _ = eng.train_classical(enc, labels)
    view = enc[skip:]
    pops = torch.empty((rows - skip, C), dtype=torch.int32, device=enc.device)
    pred = eng.predict(cv, view, popcounts=pops)
    eng.dc.check()
    encn = view.cpu().numpy().view(np.uint32)
    cvn = cv.cpu().numpy().view(np.uint32)
    eb, cb = O.unpack_rows(encn, D), O.unpack_rows(cvn, D)
    ref = (eb[:, None, :] != cb[None, :, :]).sum(-1)
    np.testing.assert_array_equal(pops.cpu().numpy(), ref)
    m = O.NaiveModel(C, D, cbk.model_tiebreak.cpu().numpy().view(np.uint32))
    m.cv[:] = cb
    ol, _ = m.predict(encn)
    np.testing.assert_array_equal(pred.cpu().numpy(), ol)


@pytest.mark.parametrize("D", [65536, 4096 + 64])
def test_device_predict_many_classes_extreme_counts(D):
    """Dot products up to D (all-ones rows against all-ones classes) and 0
    stay exact through the tensor-core scan's f32 accumulators."""
    from paper_2206_04746_b200 import device as dv
    C, rows, W = 64, 300, D // 32
    cbk = dv.DeviceCodebook.make(8, 16, D, seed=5)
    eng = dv.Engine(cbk, C)
    rng = np.random.default_rng(D)
    encn = rng.integers(0, 2**32, (rows, W), dtype=np.uint64).astype(np.uint32)
    encn[::3] = 0xFFFFFFFF
    encn[1::7] = 0
    cvn = rng.integers(0, 2**32, (C, W), dtype=np.uint64).astype(np.uint32)
    cvn[::2] = 0xFFFFFFFF
    cvn[5] = 0
    enc = torch.from_numpy(encn.view(np.int32)).cuda()
    cv = torch.from_numpy(cvn.view(np.int32)).cuda()
    pops = torch.empty((rows, C), dtype=torch.int32, device="cuda")
    pred = eng.predict(cv, enc, popcounts=pops)
    eng.dc.check()
    eb, cb = O.unpack_rows(encn, D), O.unpack_rows(cvn, D)
    ref = (eb[:, None, :] != cb[None, :, :]).sum(-1)
    np.testing.assert_array_equal(pops.cpu().numpy(), ref)
    key = ref.astype(np.int64) * C + np.arange(C)[None, :]
    np.testing.assert_array_equal(pred.cpu().numpy(), key.argmin(1))


@pytest.mark.parametrize("C,D,rows,bsz", [(100, 32768, 3000, 1024), (64, 10000, 2600, 512)])
def test_online_tensor_core_scoring_matches_popc_scoring(C, D, rows, bsz, monkeypatch):
    """Many-class online training scores each batch on the tensor cores
    (split-K tcgen05 popcounts feeding the persistent trainer); it must give
    the same fp64 accumulators, weights and class vectors as the POPC-scored
    persistent kernel (HVB200_ONLINE_TC=0)."""
    from paper_2206_04746_b200 import device as dv
    cbk = dv.DeviceCodebook.make(64, 16, D, seed=3)
    eng = dv.Engine(cbk, C)
    bins8, labels = eng.synth(0, rows, 0, 5)
    enc = eng.encode(bins8)
    tc = eng.train_online(enc, labels, bsz)
    monkeypatch.setenv("HVB200_ONLINE_TC", "0")
    ref = eng.train_online(enc, labels, bsz)
    eng.dc.check()
    for a, b in zip(tc, ref):
        assert torch.equal(a, b)


def test_device_online_delta_mode_emulated_ranks():
    """Data-parallel delta mode emulated with 2 ranks on one
    GPU: each rank's per-class deltas for its slice of a batch are summed (the
    all-reduce) and applied. One batch from identical state must give
    accumulators within 1e-12 relative of the exact in-place trainer; class
    bits may differ only where 2*acc == weight up to rounding (a tie the
    reference itself resolves by its own rounding order)."""
    from paper_2206_04746_b200 import device as dv
    import paper_2206_04746_b200._native as N
    F, B, D, C, bsz = 561, 16, 10000, 6, 512
    cbk = dv.DeviceCodebook.make(F, B, D, seed=4)
    eng = dv.Engine(cbk, C)
    bins8, labels = eng.synth(0, bsz, 0, 7)
    enc = eng.encode(bins8)
    acc_x, w_x, c_x, cv_x = eng.train_online(enc, labels, bsz)  # bootstrap + one online batch
    world = 2
    counts, crow = eng.zero_counts()
    eng.class_counts(enc, labels, counts, crow)
    acc = counts[:, :D].to(torch.float64).contiguous()
    weight = crow.to(torch.float64)
    cnt = crow.clone()
    cv = eng.binarize(counts, crow)
    tot = None
    for r in range(world):
        lo, hi = dv.online_slice(0, bsz, r, world)
        d = [torch.empty_like(acc), torch.empty_like(weight), torch.empty_like(cnt),
             torch.empty(C, dtype=torch.int32, device=acc.device)]
        N.check(N.lib().hv_dev_online_delta(eng.dc.h, dv._ptr(cv), C, D, dv._ptr(enc[lo:hi]), hi - lo,
                                            dv._ptr(labels[lo:hi]), 1.0, *[dv._ptr(t) for t in d]))
        tot = d if tot is None else [a + b for a, b in zip(tot, d)]
    N.check(N.lib().hv_dev_apply_online_delta(eng.dc.h, C, D, *[dv._ptr(t) for t in tot],
                                              dv._ptr(cbk.model_tiebreak), dv._ptr(acc), dv._ptr(weight),
                                              dv._ptr(cnt), dv._ptr(cv)))
    eng.dc.check()
    torch.cuda.synchronize()
    rel = ((acc - acc_x).abs() / acc_x.abs().clamp_min(1.0)).max().item()
    assert rel <= 1e-12, rel
    assert ((weight - w_x).abs() / w_x).max().item() <= 1e-12
    assert torch.equal(cnt, c_x)
    diff = (cv ^ cv_x).cpu().numpy().view(np.uint32)
    bits = O.unpack_rows(diff, D).astype(bool)
    margin = (2.0 * acc_x - w_x[:, None]).abs().cpu().numpy()
    assert np.all(margin[bits] <= 1e-9 * w_x.cpu().numpy()[np.nonzero(bits)[0]]), "flip away from a tie"


@pytest.mark.parametrize("F,D,C,rows,bsz,world", [(561, 10000, 6, 3000, 256, 2), (561, 10000, 6, 1500, 1, 3),
                                                  (342, 1000, 2, 2000, 1024, 3), (617, 10000, 26, 2000, 100, 8)])
def test_dsliced_online_emulated_ranks_bitexact(F, D, C, rows, bsz, world):
    """Exact multi-GPU online training (device.DSlicedOnline) with `world`
    ranks emulated on one GPU: each rank encodes only its word slice, the
    per-batch partial popcounts are summed (the all-reduce), and the stitched
    accumulators / class vectors / weights are bit-identical to the
    single-GPU exact trainer (itself bit-exact vs the reference)."""
    from paper_2206_04746_b200 import device as dv
    cbk = dv.DeviceCodebook.make(F, 16, D, seed=F + world)
    eng = dv.Engine(cbk, C)
    bins8, labels = eng.synth(0, rows, 0, 7)
    enc = eng.encode(bins8)
    acc_x, w_x, c_x, cv_x = eng.train_online(enc, labels, bsz)
    W = enc.shape[1]
    ranks = []
    for r in range(world):
        w0, nw = dv.word_slice(W, r, world)
        sl = eng.encode_words(bins8, w0, nw)
        assert torch.equal(sl, enc[:, w0:w0 + nw])
        ranks.append(dv.DSlicedOnline(eng, sl, labels, bsz, w0))
    for start, n in ranks[0].batches():
        tot = sum(rk.partial(start, n).clone() for rk in ranks)
        for rk in ranks:
            rk.update(start, n, tot)
    eng.dc.check()
    torch.cuda.synchronize()
    assert torch.equal(torch.cat([rk.acc for rk in ranks], dim=1), acc_x)
    assert torch.equal(torch.cat([rk.cv for rk in ranks], dim=1), cv_x)
    for rk in ranks:
        assert torch.equal(rk.weight, w_x) and torch.equal(rk.counts, c_x)


def test_encode_words_slices_and_generic_fallback():
    """hv_dev_encode_words for id-level (fused path) and permutation (whole-row
    scratch + slice copy) equals the matching columns of a full encode."""
    from paper_2206_04746_b200 import device as dv
    import paper_2206_04746_b200._native as N
    for binding in (N.BIND_ID_LEVEL, N.BIND_PERMUTATION):
        cbk = dv.DeviceCodebook.make(100, 16, 2000, seed=9, binding=binding)
        eng = dv.Engine(cbk, 2)
        bins8, _ = eng.synth(0, 333, 0, 3)
        full = eng.encode(bins8)
        for w0, nw in [(0, 63), (5, 1), (17, 46), (62, 1)]:
            assert torch.equal(eng.encode_words(bins8, w0, nw), full[:, w0:w0 + nw]), (binding, w0, nw)


def test_peer_counts_emulated_ranks_equal_allreduce():
    """Classical counts fused with their all-reduce over peer memory
    (device.PeerCounts, csrc/hv_peer.cu) with 3 ranks emulated in one process:
    every rank's buffer ends with exactly the global counts, over several
    epochs (parity reuse after release)."""
    from paper_2206_04746_b200 import device as dv
    F, B, D, C, rows, world = 342, 16, 1000, 3, 5000, 3
    cbk = dv.DeviceCodebook.make(F, B, D, seed=2)
    eng = dv.Engine(cbk, C)
    bufs = [torch.zeros(dv.PeerCounts.buffer_bytes(eng, world), dtype=torch.uint8, device="cuda")
            for _ in range(world)]
    bases = [b.data_ptr() for b in bufs]
    pcs = [dv.PeerCounts(eng, r, world, local_ranks=bases) for r in range(world)]
    for epoch_seed in (7, 8, 9):
        bins8, labels = eng.synth(0, rows, 0, epoch_seed)
        enc = eng.encode(bins8)
        want_c, want_r = eng.zero_counts()
        eng.class_counts(enc, labels, want_c, want_r)
        spans = [dv.shard_range(rows, r, world) for r in range(world)]
        eps = [pcs[r].count(enc[lo:hi], labels[lo:hi]) for r, (lo, hi) in enumerate(spans)]
        for r in range(world):
            got_c, got_r = pcs[r].wait(eps[r])
            eng.dc.check()
            torch.cuda.synchronize()
            assert torch.equal(got_c, want_c), (epoch_seed, r)
            assert torch.equal(got_r, want_r), (epoch_seed, r)
        for r in range(world):
            pcs[r].release(eps[r])


def test_dsliced_online_fused_peer_popcounts_bitexact():
    """Word-sliced online training with the per-batch popcount all-reduce fused
    into the partial kernel over peer memory (device.PeerPopc), 3 ranks
    emulated in one process: bit-identical to the single-GPU exact trainer."""
    from paper_2206_04746_b200 import device as dv
    F, D, C, rows, bsz, world = 561, 10000, 6, 1500, 128, 3
    cbk = dv.DeviceCodebook.make(F, 16, D, seed=11)
    eng = dv.Engine(cbk, C)
    bins8, labels = eng.synth(0, rows, 0, 7)
    enc = eng.encode(bins8)
    acc_x, w_x, c_x, cv_x = eng.train_online(enc, labels, bsz)
    W = enc.shape[1]
    bufs = [torch.zeros(dv.PeerPopc.buffer_bytes(eng, bsz, world), dtype=torch.uint8, device="cuda")
            for _ in range(world)]
    bases = [b.data_ptr() for b in bufs]
    ranks, peers = [], []
    for r in range(world):
        w0, nw = dv.word_slice(W, r, world)
        ranks.append(dv.DSlicedOnline(eng, eng.encode_words(bins8, w0, nw), labels, bsz, w0))
        peers.append(dv.PeerPopc(eng, r, world, bsz, local_ranks=bases))
    for b, (start, n) in enumerate(ranks[0].batches()):
        for rk, pp in zip(ranks, peers):
            rk.peer_partial(pp, start, n, b + 1)
        for rk, pp in zip(ranks, peers):
            rk.peer_update(pp, start, n, b + 1)
    eng.dc.check()
    torch.cuda.synchronize()
    assert torch.equal(torch.cat([rk.acc for rk in ranks], dim=1), acc_x)
    assert torch.equal(torch.cat([rk.cv for rk in ranks], dim=1), cv_x)
    for rk in ranks:
        assert torch.equal(rk.weight, w_x) and torch.equal(rk.counts, c_x)


@pytest.mark.parametrize("trainer,metric,split", [("classical", 0, "tscv"), ("online", 0, "tscv"),
                                                  ("classical", 1, "subset"), ("online", 0, "subset"),
                                                  ("online", 1, "tscv")])
def test_dataset_fold_matches_reference_pipeline(trainer, metric, split):
    """run_fold_packed (experiment.cpp:148-178) on an HBM-resident fp64 dataset:
    discretizer fit on the train rows, discretize, encode, train, predict —
    labels and fitted min/max bit-identical to the oracle pipeline, for
    contiguous (time-series) and arbitrary (leave-one-out style) row subsets,
    over several folds of the same resident dataset."""
    rng = np.random.default_rng(17 + metric)
    n, F, C, B, D = 900, 37, 4, 16, 1000
    y = rng.integers(0, C, n).astype(np.int32)
    centers = rng.normal(size=(C, F))
    X = centers[y] + 0.7 * rng.normal(size=(n, F))
    X[5, 3] = np.nan
    ds = hv.Dataset(X, y)
    cb = hv.make_codebook(0, 0, F, B, D, 123)
    etb = hv.generate_random(1, D, 456)
    cfg = hv.ModelConfig(class_count=C, dim=D, metric=metric, gamma=0.8, seed=9)
    mtb = hv.generate_random(1, D, hv.derive_seed(9, 3))
    for k in range(3):
        if split == "tscv":
            tr = np.arange(0, 300 + 200 * k)
            te = np.arange(300 + 200 * k, 400 + 200 * k)
        else:
            perm = rng.permutation(n)
            tr, te = np.sort(perm[:500]), perm[500:650]
        labels, mn, mx = ds.fold(tr, te, cb, etb, cfg, trainer, 64)
        omn, omx = O.fit_discretizer(X[tr], B)
        np.testing.assert_array_equal(mn, omn)
        np.testing.assert_array_equal(mx, omx)
        bins = O.discretize_matrix(X[np.concatenate([tr, te])], omn, omx, B)
        enc = O.encode_batch(bins, cb.id_vectors.words, cb.value_vectors.words, B, D, O.BIND_ID_LEVEL, etb.words)
        m = O.NaiveModel(C, D, mtb.words, metric, 0.8)
        if trainer == "online":
            m.train_online(enc[:tr.size], y[tr], 64)
        else:
            m.train_classical(enc[:tr.size], y[tr])
        want, _ = m.predict(enc[tr.size:])
        np.testing.assert_array_equal(labels, want)
    bad = y.copy()
    bad[250] = C
    ds2 = hv.Dataset(X, bad)
    with pytest.raises(hv.InvalidArgument, match=r"online_update: label 4 at row 58 out of range \(classes = 4\)"):
        ds2.fold(np.arange(300), np.arange(300, 400), cb, etb, cfg, "online", 64)
    with pytest.raises(hv.InvalidArgument, match=r"train_classical: label 4 at row 250 out of range"):
        ds2.fold(np.arange(300), np.arange(300, 400), cb, etb, cfg, "classical", 64)
    with pytest.raises(hv.InvalidArgument, match="fit_discretizer: empty training matrix"):
        ds.fold(np.arange(0), np.arange(10), cb, etb, cfg)
    ds.close()
    ds2.close()
