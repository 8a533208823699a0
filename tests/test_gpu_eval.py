"""GPU parity for the evaluation tail of an experiment (eval.cpp:12-116,
experiment.cpp:280-345): label smoothing, sample metrics and episode counts
computed on the device, against the reference's golden outputs and the C
oracle; and the HBM-resident experiment (folds -> concatenation -> smoothing
-> metrics) against the oracle pipeline. Counts and labels bit-exact; ratios
bit-exact (the same double expressions on exact counts)."""
import numpy as np
import pytest

import oracle_ref as O
from golden_io import Case, cases

pytestmark = pytest.mark.gpu

hv = pytest.importorskip("paper_2206_04746_b200.hypervec")
from paper_2206_04746_b200 import launch_count  # noqa: E402


def _bits(x):
    return np.array([np.nan if x is None else x], np.float64).view(np.uint64)[0]


def _check_report(r, counts, ratios):
    assert [r.tp, r.fp, r.tn, r.fn] == [int(v) for v in counts[:4]]
    for got, want in zip((r.accuracy, r.tpr, r.ppv, r.f1), ratios):
        assert _bits(got) == np.array([want], np.float64).view(np.uint64)[0], (got, want)


@pytest.mark.parametrize("name", cases("eval_"))
def test_eval_matches_reference_goldens(name):
    c = Case(name)
    pred, truth, pos = c["pred"], c["truth"], c.int("positive")
    before = launch_count()
    for w in (1, 3, 5, 9, 31, 101):
        if c.has(f"smooth_{w}"):
            np.testing.assert_array_equal(hv.smooth_labels(pred, w), c[f"smooth_{w}"])
    e = hv.episode_metrics(pred, truth, pos)
    assert [e.detected, e.total, e.false_positive] == [int(v) for v in c["episodes"]]
    if len(pred):
        _check_report(hv.sample_metrics(pred, truth, pos), c["counts"], c["ratios"])
        assert launch_count() > before


@pytest.mark.parametrize("n,window", [(1, 3), (2, 3), (5, 99), (1_000_003, 1), (1_000_003, 9), (4_000_000, 241)])
def test_smoothing_and_metrics_at_scale_vs_oracle(n, window):
    rng = np.random.default_rng(n + window)
    # seizure-like truth: rare positive runs; predictions with glitches
    truth = (np.cumsum(rng.random(n) < 0.004) % 2).astype(np.int32)
    pred = np.where(rng.random(n) < 0.08, 1 - truth, truth).astype(np.int32)
    np.testing.assert_array_equal(hv.smooth_labels(pred, window), O.smooth_labels(pred, window))
    counts, ratios = O.sample_metrics(pred, truth, 1)
    _check_report(hv.sample_metrics(pred, truth, 1), counts, ratios)
    for pos in (0, 1):
        e = hv.episode_metrics(pred, truth, pos)
        assert [e.detected, e.total, e.false_positive] == list(O.episode_metrics(pred, truth, pos))


def test_eval_edge_cases_and_reference_messages():
    # test_eval.cpp:24-55 known answers
    labels = [0, 1, 0, 1, 1, 1, 0]
    assert hv.smooth_labels(labels, 3).tolist() == [0, 0, 1, 1, 1, 1, 1]
    assert hv.smooth_labels(labels, 1).tolist() == labels
    assert hv.smooth_labels(labels, 7).tolist() == [1] * 7
    assert hv.smooth_labels(labels, 99).tolist() == [1] * 7
    assert hv.smooth_labels([0, 1], 3).tolist() == [1, 1]
    assert hv.smooth_labels([], 3).size == 0
    with pytest.raises(hv.InvalidArgument, match=r"^smooth_labels: window must be odd and >= 1, got 2$"):
        hv.smooth_labels([0, 1], 2)
    with pytest.raises(hv.InvalidArgument, match=r"^smooth_labels: window must be odd and >= 1, got 0$"):
        hv.smooth_labels([0, 1], 0)
    with pytest.raises(hv.InvalidArgument, match=r"^smooth_labels: non-binary label 2 at index 1$"):
        hv.smooth_labels([0, 2, 0, 5], 3)
    with pytest.raises(hv.InvalidArgument, match=r"^sample_metrics: 2 predictions vs 1 labels$"):
        hv.sample_metrics([1, 0], [1], 1)
    with pytest.raises(hv.InvalidArgument, match=r"^sample_metrics: empty sequences$"):
        hv.sample_metrics([], [], 1)
    with pytest.raises(hv.InvalidArgument, match=r"^episode_metrics: 1 predictions vs 2 labels$"):
        hv.episode_metrics([1], [1, 0], 1)
    # test_eval.cpp:106-115: undefined ratios stay absent
    r = hv.sample_metrics([0, 0], [0, 0], 1)
    assert r.accuracy == 1.0 and r.tpr is None and r.ppv is None and r.f1 is None
    # test_eval.cpp:128-148 episode counts
    e = hv.episode_metrics([], [], 1)
    assert (e.detected, e.total, e.false_positive) == (0, 0, 0)
    pred = [1, 0, 0, 0, 0, 0, 1, 1, 0, 0]
    truth = [1, 1, 0, 1, 1, 0, 0, 0, 1, 0]
    e = hv.episode_metrics(pred, truth, 1)
    assert [e.detected, e.total, e.false_positive] == list(O.episode_metrics(pred, truth, 1))


def _oracle_fold(X, y, tr, te, cb, etb, mtb, C, B, D, trainer, metric, gamma, batch):
    omn, omx = O.fit_discretizer(X[tr], B)
    bins = O.discretize_matrix(X[np.concatenate([tr, te])], omn, omx, B)
    enc = O.encode_batch(bins, cb.id_vectors.words, cb.value_vectors.words, B, D, O.BIND_ID_LEVEL, etb.words)
    m = O.NaiveModel(C, D, mtb.words, metric, gamma)
    if trainer == "online":
        m.train_online(enc[:tr.size], y[tr], batch)
    else:
        m.train_classical(enc[:tr.size], y[tr])
    return m.predict(enc[tr.size:])[0]


@pytest.mark.parametrize("C,trainer,window", [(2, "classical", 5), (2, "online", 9), (2, "classical", 1),
                                              (3, "classical", 5)])
def test_resident_experiment_matches_oracle_protocol(C, trainer, window):
    """run_experiment with a time-series split: predictions of every fold stay
    in HBM, are concatenated in row order, smoothed (binary runs only) and
    scored on the device; the oracle replays the same folds on the CPU."""
    rng = np.random.default_rng(40 + C)
    n, F, B, D = 1200, 24, 16, 2048
    if C == 2:
        y = (np.cumsum(rng.random(n) < 0.02) % 2).astype(np.int32)
    else:
        y = rng.integers(0, C, n).astype(np.int32)
    centers = rng.normal(size=(C, F))
    X = centers[y] + 1.3 * rng.normal(size=(n, F))
    ds = hv.Dataset(X, y)
    cb = hv.make_codebook(0, 0, F, B, D, 321)
    etb = hv.generate_random(1, D, 654)
    cfg = hv.ModelConfig(class_count=C, dim=D, metric=0, gamma=1.0, seed=11)
    mtb = hv.generate_random(1, D, hv.derive_seed(11, 3))
    ex = ds.experiment()
    predicted = np.full(n, -1, np.int32)
    # tscv-like: expanding train window, next block tested; one block re-tested (last fold wins)
    folds = [(np.arange(0, 300), np.arange(300, 500)), (np.arange(0, 500), np.arange(500, 800)),
             (np.arange(0, 800), np.arange(800, 1000)), (np.arange(0, 700), np.arange(700, 800)),
             # rows listed twice in one fold (both copies get the same label, as in the reference loop)
             (np.arange(0, 350), np.concatenate([np.arange(1100, 1200), np.arange(1150, 1200)[::-1]]))]
    for tr, te in folds:
        ex.fold(tr, te, cb, etb, cfg, trainer, 64)
        for r, lab in zip(te, _oracle_fold(X, y, tr, te, cb, etb, mtb, C, B, D, trainer, 0, 1.0, 64)):
            predicted[r] = lab  # experiment.cpp:307-309 order
    res = ex.finish(C, window, 1)
    tested = np.nonzero(predicted >= 0)[0]
    pred_seq, truth_seq = predicted[tested], y[tested]
    final = O.smooth_labels(pred_seq, window) if (C == 2 and window > 1) else pred_seq
    assert res.fold_count == 5
    np.testing.assert_array_equal(res.rows, tested)
    np.testing.assert_array_equal(res.truth, truth_seq)
    np.testing.assert_array_equal(res.predicted, pred_seq)
    np.testing.assert_array_equal(res.final, final)
    counts, ratios = O.sample_metrics(final, truth_seq, 1)
    _check_report(res.report, counts, ratios)
    ep = O.episode_metrics(final, truth_seq, 1)
    e = res.report.episodes
    assert [e.detected, e.total, e.false_positive] == list(ep)
    ex.close()
    empty = ds.experiment()
    with pytest.raises(hv.InvalidArgument, match="no test samples produced by split"):
        empty.finish(C, window, 1)
    ds.close()


def test_gpu_results_save_byte_identical_to_reference_files():
    """§8 f4: hypervectors encoded and models trained on the B200, written
    with the HVPB/HVMD containers, are the reference's files byte for byte."""
    from paper_2206_04746_b200 import containers as cio

    c, p = Case("containers"), Case("pipeline_odd")
    F, D, C, tr = 13, 1000, 3, 125
    cb = hv.make_codebook(0, 0, F, 16, D, hv.derive_seed(12, 1))
    etb = hv.generate_random(1, D, hv.derive_seed(12, 2))
    enc = hv.encode_batch(p["bins"], 157, cb, etb)
    assert cio.write_packed(enc) == bytes(c["hvpb_encoded"].astype(np.uint8))
    assert cio.save_codebook(cb) == bytes(c["hvcb_random"].astype(np.uint8))
    train = hv.PackedBitMatrix(tr, D, enc.words[:tr])
    cfg = hv.ModelConfig(class_count=C, dim=D, metric=0, gamma=0.6, seed=12)
    y = p["y"][:tr]
    assert cio.save_model(hv.train_classical(train, y, cfg)) == bytes(c["hvmd_classical"].astype(np.uint8))
    assert cio.save_model(hv.train_online(train, y, 5, cfg)) == bytes(c["hvmd_online_b5"].astype(np.uint8))
    # and a reference file loads into a model the GPU predicts with
    m = cio.load_model(bytes(c["hvmd_classical"].astype(np.uint8)))
    labels, _ = hv.predict_arrays(m, hv.PackedBitMatrix(157 - tr, D, enc.words[tr:]))
    np.testing.assert_array_equal(labels, p["classical_pred"])
