"""Parity at BASELINE.json's full sizes (CHB-MIT 7.06 M rows; Large 10 M rows,
D = 32768, 100 classes) through properties the oracle can check in seconds:

* sampled rows spread over the whole dataset (first, last, and random) are
  re-derived on the CPU — bins by the C synth generator, hypervectors by the
  oracle's byte-per-bit encoder — and must equal the device's words;
* the classical counts of every train row are recounted independently with
  torch bit ops (chunked), and the class vectors must equal the oracle's
  majority_binarize of those counts with the model tiebreak;
* the predictions (labels and fp64 distances) of sampled test rows must equal
  the oracle's predict against the same class vectors;
* online training of a 256-batch prefix is bit-exact against the oracle.

These are the bench workloads themselves, not scaled-down stand-ins."""
import numpy as np
import pytest
import torch

import oracle_ref as O

pytestmark = pytest.mark.gpu

dv = pytest.importorskip("paper_2206_04746_b200.device")


def _u32(t):
    return t.cpu().numpy().view(np.uint32)


def _sample(n, k, seed):
    rng = np.random.default_rng(seed)
    idx = np.unique(np.concatenate([[0, 1, n // 2, n - 2, n - 1], rng.integers(0, n, k)]))
    return idx


def _check_sampled_encodes(eng, cbk, bins8, enc, idx, C, label_kind, data_seed):
    F, B, D = cbk.features, cbk.bins, cbk.dim
    ref_bins = np.concatenate([O.synth_c(int(r), 1, F, C, B, label_kind, data_seed)[0] for r in idx])
    np.testing.assert_array_equal(bins8[torch.as_tensor(idx, device=bins8.device)][:, :F].cpu().numpy(), ref_bins)
    want = O.encode_batch(ref_bins, _u32(cbk.id_vectors), _u32(cbk.value_vectors), B, D, O.BIND_ID_LEVEL,
                          _u32(cbk.encode_tiebreak))
    np.testing.assert_array_equal(_u32(enc[torch.as_tensor(idx, device=enc.device)]), want)


def _torch_class_counts(enc, labels, C, D, chunk=65536):
    """Independent recount: unpack every row's bits with torch and sum per class
    (labels outside [0, C) are skipped)."""
    W = enc.shape[1]
    shifts = torch.arange(32, device=enc.device, dtype=torch.int32)
    out = torch.zeros((C, 32 * W), dtype=torch.int64, device=enc.device)
    for r0 in range(0, enc.shape[0], chunk):
        e = enc[r0:r0 + chunk]
        bits = ((e.unsqueeze(-1) >> shifts) & 1).to(torch.uint8).reshape(e.shape[0], 32 * W)
        y = labels[r0:r0 + chunk].long()
        for c in range(C):
            m = y == c
            if m.any():
                out[c] += bits[m].sum(0, dtype=torch.int64)
    return out[:, :D]


def _check_classical_and_predict(eng, cbk, enc, labels, ntr, C, test_idx):
    D = cbk.dim
    cv, counts, rows = eng.train_classical(enc[:ntr], labels[:ntr])
    torch.cuda.synchronize()
    want_rows = torch.bincount(labels[:ntr].long(), minlength=C)
    assert torch.equal(rows.cpu(), want_rows.cpu())
    if C <= 10:
        recount = _torch_class_counts(enc[:ntr], labels[:ntr], C, D)
        assert torch.equal(counts[:, :D].long(), recount)
    else:  # Large: recount a class subset (all rows still stream through)
        sub = torch.tensor([0, 1, 37, C - 1], device=enc.device)
        lab = labels[:ntr].long()
        remap = torch.full((C,), len(sub), dtype=torch.long, device=enc.device)
        remap[sub] = torch.arange(len(sub), device=enc.device)
        recount = _torch_class_counts(enc[:ntr], remap[lab].int(), len(sub), D)
        assert torch.equal(counts[sub][:, :D].long(), recount)
    cnt = counts.cpu().numpy().astype(np.uint64)
    tb = _u32(cbk.model_tiebreak)
    ncls = rows.cpu().numpy()
    tb_bits = O.unpack_rows(tb.reshape(1, -1), D).reshape(-1)
    for c in range(C):  # an empty class binarises to the tiebreak (2*0 == 0)
        want = O.pack_rows(O.majority_binarize(cnt[c, :D], int(ncls[c]), tb_bits).reshape(1, -1))
        np.testing.assert_array_equal(_u32(cv[c]).reshape(1, -1), want)
    # predictions of sampled test rows against the same class vectors
    test = enc[ntr:]
    dist = torch.empty((test.shape[0], C), dtype=torch.float64, device=enc.device)
    lab = eng.predict(cv, test, distances=dist)
    m = O.NaiveModel(C, D, tb)
    m.cv = O.unpack_rows(_u32(cv), D).copy()
    ti = torch.as_tensor(test_idx, device=enc.device)
    ol, od = m.predict(_u32(test[ti]))
    np.testing.assert_array_equal(lab[ti].cpu().numpy(), ol)
    np.testing.assert_array_equal(dist[ti].cpu().numpy().view(np.uint64), od.view(np.uint64))
    return cv


def test_chbmit_full_size_encode_train_predict_online():
    """BASELINE configs[3]: 7.06 M CHB-MIT-shaped rows (F = 342, D = 10000, 2 unbalanced classes)."""
    N, F, B, D, C = 7_060_000, 342, 16, 10000, 2
    cbk = dv.DeviceCodebook.make(F, B, D, seed=20)
    eng = dv.Engine(cbk, C)
    bins8, labels = eng.synth(0, N, 1, 9)
    enc = eng.encode(bins8)
    torch.cuda.synchronize()
    _check_sampled_encodes(eng, cbk, bins8, enc, _sample(N, 40, 1), C, 1, 9)
    ntr = N * 4 // 5
    _check_classical_and_predict(eng, cbk, enc, labels, ntr, C, _sample(N - ntr, 3000, 2))
    # online: a 256-batch prefix (262,144 rows) bit-exact against the oracle
    pre = 256 * 1024
    acc, weight, counts, cv = eng.train_online(enc[:pre], labels[:pre], 1024)
    om = O.NaiveModel(C, D, _u32(cbk.model_tiebreak)).train_online(_u32(enc[:pre]), labels[:pre].cpu().numpy(), 1024)
    assert torch.equal(acc.cpu(), torch.from_numpy(om.acc))
    np.testing.assert_array_equal(_u32(cv), om.class_vectors)


def test_large_full_size_encode_train_predict():
    """BASELINE configs[4]: 10 M rows, F = 617, D = 32768, 100 classes (tcgen05 prediction)."""
    N, F, B, D, C = 10_000_000, 617, 16, 32768, 100
    cbk = dv.DeviceCodebook.make(F, B, D, seed=21)
    eng = dv.Engine(cbk, C)
    bins8, labels = eng.synth(0, N, 0, 5)
    enc = eng.encode(bins8)
    torch.cuda.synchronize()
    _check_sampled_encodes(eng, cbk, bins8, enc, _sample(N, 12, 3), C, 0, 5)
    del bins8
    ntr = N * 4 // 5
    _check_classical_and_predict(eng, cbk, enc, labels, ntr, C, _sample(N - ntr, 1000, 4))


def test_chbmit_full_size_online_two_exact_paths_agree():
    """The whole CHB-MIT online run (5.65 M train rows, 5,516 batches of 1,024)
    through two independent exact implementations — the persistent single-GPU
    trainer and the word-sliced multi-GPU mode with 2 ranks emulated on this
    GPU (different kernels: slice init, partial popcounts summed across ranks,
    slice update) — must give bit-identical fp64 accumulators, weights, counts
    and class vectors (model.cpp:250-301). The 256-batch prefix is pinned
    against the oracle in the test above."""
    N, F, B, D, C = 7_060_000, 342, 16, 10000, 2
    ntr = N * 4 // 5
    cbk = dv.DeviceCodebook.make(F, B, D, seed=20)
    eng = dv.Engine(cbk, C)
    bins8, labels = eng.synth(0, ntr, 1, 9)
    enc = eng.encode(bins8)
    acc, weight, counts, cv = eng.train_online(enc, labels, 1024)
    del enc
    W = eng.W
    ranks = []
    for r in range(2):
        w0, nw = dv.word_slice(W, r, 2)
        ranks.append(dv.DSlicedOnline(eng, eng.encode_words(bins8, w0, nw), labels, 1024, w0))
    for start, n in ranks[0].batches():
        tot = ranks[0].partial(start, n).clone()
        tot += ranks[1].partial(start, n)
        for rk in ranks:
            rk.update(start, n, tot)
    eng.dc.check()
    torch.cuda.synchronize()
    assert torch.equal(torch.cat([rk.acc for rk in ranks], dim=1), acc)
    assert torch.equal(torch.cat([rk.cv for rk in ranks], dim=1), cv)
    for rk in ranks:
        assert torch.equal(rk.weight, weight) and torch.equal(rk.counts, counts)
