"""Pin the C oracle against golden vectors produced by the reference library.

The fixtures in tests/golden/cases were written by oracle/golden_gen.cpp linked
against the reference's own sources (oracle/_ref/libhypervec.a). Passing these
is what entitles the oracle to serve as the parity checker for the GPU engine.
"""
import numpy as np
import pytest

import oracle_ref as O
from golden_io import Case, cases


def test_mt19937_64_and_substreams():
    c = Case("rng")
    for seed in (0, 1, 42, 0xDEADBEEFCAFEF00D):
        np.testing.assert_array_equal(O.mt64(seed, 700), c[f"mt64_{seed}"])
    sm = [O.splitmix64((x * 0x9E3779B97F4A7C15) & ((1 << 64) - 1)) for x in range(64)]
    np.testing.assert_array_equal(np.array(sm, np.uint64), c["splitmix64"])
    ds = np.array([[O.derive_seed(x, t) for t in range(1, 5)] for x in range(64)], np.uint64)
    np.testing.assert_array_equal(ds, c["derive_seed"])


def test_codebook_generators():
    c = Case("codebook")
    np.testing.assert_array_equal(O.generate_random(5, 10240, 99), c["random_5x10240_s99"])
    np.testing.assert_array_equal(O.generate_random(3, 33, 7), c["random_3x33_s7"])
    np.testing.assert_array_equal(O.generate_scale_random(16, 10240, 7), c["scale_random_16x10240_s7"])
    np.testing.assert_array_equal(O.generate_scale_random(17, 32, 1), c["scale_random_17x32_s1"])
    np.testing.assert_array_equal(O.generate_sandwich(8, 1000, 5), c["sandwich_8x1000_s5"])
    np.testing.assert_array_equal(O.generate_sandwich(5, 64, 3), c["sandwich_5x64_s3"])
    for gi, g in enumerate(("random", "scale_random", "sandwich")):
        idv, val = O.make_codebook(gi, 12, 8, 1024, 77)
        np.testing.assert_array_equal(idv, c[f"cb_{g}_id"])
        np.testing.assert_array_equal(val, c[f"cb_{g}_value"])
    with pytest.raises(ValueError):
        O.generate_scale_random(17, 31, 1)
    with pytest.raises(ValueError):
        O.generate_sandwich(4, 999, 5)


@pytest.mark.parametrize("name", cases("kernels_"))
def test_bit_kernels(name):
    c = Case(name)
    d = c.int("dim")
    a, b, b1 = c["a"], c["b"], c["b1"]
    np.testing.assert_array_equal(O.pack_rows(a), c["pack_a"])
    np.testing.assert_array_equal(O.unpack_rows(c["pack_a"], d), a)
    np.testing.assert_array_equal(O.pack_rows(O.xor_bind(a, b)), c["xor_ab"])
    np.testing.assert_array_equal(O.pack_rows(O.xor_bind(a, b1)), c["xor_ab1"])
    for k, s in enumerate(c["shifts"]):
        np.testing.assert_array_equal(O.pack_rows(O.rotate(a, int(s))), c[f"rot_{k}"])
    np.testing.assert_array_equal(O.horizontal_sum(a), c["hsum"])
    np.testing.assert_array_equal(O.pack_rows(O.transpose(a)), c["transpose"])
    np.testing.assert_array_equal(O.vertical_sum(a), c["vsum"])
    got = O.majority_binarize(c["maj_counts"], c.int("maj_n"), c["maj_tiebreak"])
    np.testing.assert_array_equal(O.pack_rows(got[None, :]), c["maj_out"])


def test_discretizer():
    c = Case("discretize")
    mn, mx = O.fit_discretizer(c["data"], 16)
    np.testing.assert_array_equal(mn, c["min"])
    np.testing.assert_array_equal(mx, c["max"])
    np.testing.assert_array_equal(O.discretize_matrix(c["data"], mn, mx, 16), c["bins"])
    np.testing.assert_array_equal(O.discretize_matrix(c["probe"], mn, mx, 16), c["probe_bins"])


@pytest.mark.parametrize("name", cases("encode_"))
def test_encode(name):
    c = Case(name)
    F, B, D = c.int("F"), c.int("B"), c.int("D")
    idv, val = O.make_codebook(c.int("generation"), F, B, D, c.int("seed"))
    tb = O.generate_random(1, D, c.int("tiebreak_seed"))
    got = O.encode_batch(c["bins"], idv, val, B, D, c.int("binding"), tb)
    np.testing.assert_array_equal(got, c["out"])


@pytest.mark.parametrize("name", cases("pipeline_"))
def test_pipeline(name):
    c = Case(name)
    n, F, C, D = c.int("rows"), c.int("features"), c.int("classes"), c.int("dim")
    seed, ntr = c.int("seed"), c.int("train_rows")
    gamma = c.float_bits("gamma_bits")
    mn, mx = O.fit_discretizer(c["X"][:ntr], 16)
    np.testing.assert_array_equal(mn, c["min"])
    np.testing.assert_array_equal(mx, c["max"])
    bins = O.discretize_matrix(c["X"], mn, mx, 16)
    np.testing.assert_array_equal(bins, c["bins"])
    idv, val = O.make_codebook(O.GEN_RANDOM, F, 16, D, O.derive_seed(seed, 1))
    etb = O.generate_random(1, D, O.derive_seed(seed, 2))
    enc = O.encode_batch(bins, idv, val, 16, D, O.BIND_ID_LEVEL, etb)
    np.testing.assert_array_equal(enc, c["encoded"])
    mtb = O.generate_random(1, D, O.derive_seed(seed, 3))
    np.testing.assert_array_equal(mtb, c["model_tiebreak"])
    y = c["y"]
    train, test = enc[:ntr], enc[ntr:]

    m = O.NaiveModel(C, D, mtb, O.HAMMING, gamma).train_classical(train, y[:ntr])
    np.testing.assert_array_equal(m.acc, c["classical_acc"])
    np.testing.assert_array_equal(m.weight, c["classical_weight"])
    np.testing.assert_array_equal(m.counts, c["classical_counts"])
    np.testing.assert_array_equal(m.class_vectors, c["classical_cv"])
    labels, dist = m.predict(test)
    np.testing.assert_array_equal(labels, c["classical_pred"])
    np.testing.assert_array_equal(dist, c["classical_dist"])

    for bsz in c["batch_sizes"]:
        k = f"online_b{int(bsz)}"
        on = O.NaiveModel(C, D, mtb, O.HAMMING, gamma).train_online(train, y[:ntr], int(bsz))
        # The oracle keeps the reference's per-element, sample-ordered fp64
        # adds, so it is bit-identical to the packed reference.
        np.testing.assert_array_equal(on.acc, c[k + "_acc"])
        np.testing.assert_array_equal(on.weight, c[k + "_weight"])
        np.testing.assert_array_equal(on.counts, c[k + "_counts"])
        np.testing.assert_array_equal(on.class_vectors, c[k + "_cv"])
        np.testing.assert_array_equal(on.predict(test)[0], c[k + "_pred"])

    cm = O.NaiveModel(C, D, mtb, O.COSINE, gamma).train_classical(train, y[:ntr])
    cl, cd = cm.predict(test)
    np.testing.assert_array_equal(cl, c["cosine_pred"])
    np.testing.assert_allclose(cd, c["cosine_dist"], rtol=1e-9, atol=0)


def test_online_update_single_batch():
    c = Case("online_update")
    C_, D = c.int("classes"), c.int("dim")
    gamma = c.float_bits("gamma_bits")
    tb = O.generate_random(1, D, O.derive_seed(c.int("seed"), 3))
    m = O.NaiveModel(C_, D, tb, O.HAMMING, gamma).train_classical(O.pack_rows(c["base"]), c["base_y"])
    m.online_update(O.pack_rows(c["batch"]), c["y"])
    np.testing.assert_array_equal(m.acc, c["acc"])
    np.testing.assert_array_equal(m.weight, c["weight"])
    np.testing.assert_array_equal(m.counts, c["counts"])
    np.testing.assert_array_equal(m.class_vectors, c["cv"])


def test_synth_generator_matches_reference_make_synth():
    """make_synth (tests/support/synth.cpp:16-47) restated with the oracle's RNG."""
    c = Case("synth")
    X, y = c["X"], c["y"]
    rows, feats, classes, grid, jitter = 64, 30, 5, 16, 0.3
    draws = O.mt64(501, rows * feats)
    unit = (draws >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    width = 1.0 / grid
    got = np.zeros((rows, feats))
    for i in range(rows):
        cls = i % classes
        for f in range(feats):
            centre = (((cls * (f + 1) + 3 * f) % grid) + 0.5) * width
            got[i, f] = centre + jitter * (2.0 * unit[i * feats + f] - 1.0) * 0.5 * width
    np.testing.assert_array_equal(y, np.arange(rows) % classes)
    np.testing.assert_array_equal(got, X)


@pytest.mark.parametrize("name", cases("eval_"))
def test_eval_smoothing_and_metrics(name):
    """eval.cpp:12-116 — smoothing, sample and episode metrics on the reference's outputs."""
    c = Case(name)
    pred, truth, pos = c["pred"], c["truth"], c.int("positive")
    for w in (1, 3, 5, 9, 31, 101):
        if c.has(f"smooth_{w}"):
            np.testing.assert_array_equal(O.smooth_labels(pred, w), c[f"smooth_{w}"])
    np.testing.assert_array_equal(O.episode_metrics(pred, truth, pos), c["episodes"])
    if len(pred):
        counts, ratios = O.sample_metrics(pred, truth, pos)
        np.testing.assert_array_equal(counts[:4], c["counts"])
        np.testing.assert_array_equal(ratios.view(np.uint64), c["ratios"].view(np.uint64))  # bit-exact, NaN = absent


def test_eval_oracle_rejects_like_reference():
    with pytest.raises(ValueError):
        O.smooth_labels([0, 1], 2)
    with pytest.raises(ValueError):
        O.smooth_labels([0, 1], 0)
    with pytest.raises(ValueError):
        O.smooth_labels([0, 2], 3)
    with pytest.raises(ValueError):
        O.sample_metrics([], [], 1)
    with pytest.raises(ValueError):
        O.sample_metrics([1, 0], [1], 1)
    # test_eval.cpp:24-32 known answers
    np.testing.assert_array_equal(O.smooth_labels([0, 1, 0, 1, 1, 1, 0], 3), [0, 0, 1, 1, 1, 1, 1])


@pytest.mark.parametrize("name", ["pipeline_small", "pipeline_odd", "pipeline_isolet"])
def test_make_synth_restatement(name):
    """The oracle's make_synth (tests/support/synth.cpp:16-47) reproduces the
    reference-written feature matrices bit for bit."""
    c = Case(name)
    X, y = O.make_synth(c.int("rows"), c.int("features"), c.int("classes"), c.int("seed"))
    np.testing.assert_array_equal(X.view(np.uint64), c["X"].view(np.uint64))
    np.testing.assert_array_equal(y, c["y"])


@pytest.mark.parametrize("name", cases("bigpipe_"))
def test_big_pipeline_inputs_and_discretizer(name):
    """The big reference pipelines store digests only: the oracle regenerates
    their inputs (make_synth -> fit_discretizer -> discretize) exactly."""
    c = Case(name)
    rows, F, ntr = c.int("rows"), c.int("features"), c.int("train_rows")
    X, y = O.make_synth(rows, F, c.int("classes"), c.int("seed"))
    np.testing.assert_array_equal(O.fnv_rows(X), c["X_fnv"])
    np.testing.assert_array_equal(y, c["y"])
    mn, mx = O.fit_discretizer(X[:ntr], 16)
    np.testing.assert_array_equal(mn, c["min"])
    np.testing.assert_array_equal(mx, c["max"])
    bins = O.discretize_matrix(X, mn, mx, 16).reshape(rows, F)
    np.testing.assert_array_equal(O.fnv_rows(bins.astype(np.uint32)), c["bins_fnv"])


def test_big_pipeline_oracle_encode_sample():
    """Sampled rows of the D = 1024 MNIST reference pipeline: the oracle's
    encoder gives the reference's encoded-row digests."""
    c = Case("bigpipe_mnist_d1k")
    rows, F, D, seed, ntr = c.int("rows"), c.int("features"), c.int("dim"), c.int("seed"), c.int("train_rows")
    X, _ = O.make_synth(rows, F, c.int("classes"), seed)
    mn, mx = O.fit_discretizer(X[:ntr], 16)
    idx = np.array([0, 1, 999, rows - 1])
    bins = O.discretize_matrix(X[idx], mn, mx, 16).reshape(len(idx), F)
    idv, val = O.make_codebook(0, F, 16, D, O.derive_seed(seed, 1))
    etb = O.generate_random(1, D, O.derive_seed(seed, 2))
    enc = O.encode_batch(bins, idv, val, 16, D, O.BIND_ID_LEVEL, etb)
    np.testing.assert_array_equal(O.fnv_rows(enc), c["encoded_fnv"][idx])
