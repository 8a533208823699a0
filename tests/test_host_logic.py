"""Host-side logic that needs no GPU: the synthetic workload definition, the
sharding plan, and the data-parallel reduction semantics (gloo, world_size 2)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle_ref as O
from paper_2206_04746_b200.device import online_slice, shard_range, shard_rows_online


@pytest.mark.parametrize("kind,classes", [(0, 26), (1, 2), (0, 5)])
def test_synth_python_matches_c(kind, classes):
    for row0 in (0, 39990, 12345678):
        b1, y1 = O.synth_bins(300, 37, classes, 16, 7, kind, start=row0)
        b2, y2 = O.synth_c(row0, 300, 37, classes, 16, kind, 7)
        np.testing.assert_array_equal(b1, b2)
        np.testing.assert_array_equal(y1, y2)


def test_synth_chbmit_imbalance():
    _, y = O.synth_c(0, 400000, 1, 2, 16, 1, 7)
    frac = y.mean()
    assert 0.002 < frac < 0.004  # ~0.3 % positives in runs of 120


def test_shard_range_covers_rows_exactly():
    for rows in (0, 1, 7, 1000, 7_060_000):
        for world in (1, 2, 3, 4, 8):
            spans = [shard_range(rows, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == rows
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))


def test_online_shards_partition_batches_in_order():
    rows, bsz = 1000, 96
    for world in (1, 2, 4, 8):
        owned = [shard_rows_online(rows, bsz, r, world) for r in range(world)]
        allrows = sorted(x for o in owned for x in o)
        assert allrows == list(range(rows))
        for o in owned:
            assert o == sorted(o)
        # rank r's slice of batch b is contiguous and ordered by rank
        for start in range(0, rows, bsz):
            n = min(bsz, rows - start)
            sl = [online_slice(start, n, r, world) for r in range(world)]
            assert sl[0][0] == start and sl[-1][1] == start + n


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _classical_worker(rank, world, port, enc, y, C, D, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = shard_range(enc.shape[0], rank, world)
    dense = O.unpack_rows(enc[lo:hi], D)
    counts = np.zeros((C, D), np.int64)
    rows = np.zeros(C, np.int64)
    for c in range(C):
        sel = y[lo:hi] == c
        counts[c] = dense[sel].sum(axis=0)
        rows[c] = sel.sum()
    tc, tr = torch.from_numpy(counts), torch.from_numpy(rows)
    dist.all_reduce(tc)
    dist.all_reduce(tr)
    if rank == 0:
        q.put((tc.numpy(), tr.numpy()))
    dist.destroy_process_group()


def test_sharded_classical_counts_allreduce_equals_full_oracle():
    """Classical training shards datapoints and all-reduces integer counts: exact."""
    rng = np.random.default_rng(3)
    C, D, n = 4, 200, 257
    enc = O.pack_rows(rng.integers(0, 2, (n, D), dtype=np.uint8))
    y = rng.integers(0, C, n).astype(np.int32)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_classical_worker, args=(r, 2, port, enc, y, C, D, q)) for r in range(2)]
    for p in procs:
        p.start()
    counts, rows = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    tb = O.generate_random(1, D, 9)
    m = O.NaiveModel(C, D, tb).train_classical(enc, y)
    np.testing.assert_array_equal(counts.astype(np.float64), m.acc)
    np.testing.assert_array_equal(rows, m.counts.astype(np.int64))


def _online_delta_reference(enc, y, C, D, bsz, gamma, world, tb):
    """NumPy restatement of the data-parallel delta-mode online trainer that
    device.Engine.train_online_sharded runs (per-rank sample-ordered deltas,
    summed across ranks, applied once per batch)."""
    dense = O.unpack_rows(enc, D).astype(np.float64)
    tbits = O.unpack_rows(tb, D)[0]
    n = enc.shape[0]
    first = min(bsz, n)
    acc = np.zeros((C, D))
    weight = np.zeros(C)
    for c in range(C):
        acc[c] = dense[:first][y[:first] == c].sum(axis=0)
        weight[c] = (y[:first] == c).sum()

    def binarize(acc, weight):
        tw = 2.0 * acc
        return np.where(tw > weight[:, None], 1, np.where(tw < weight[:, None], 0, tbits[None, :])).astype(np.uint8)

    cv = binarize(acc, weight)
    for start in range(0, n, bsz):
        m = min(bsz, n - start)
        d_acc = np.zeros((C, D))
        d_w = np.zeros(C)
        for r in range(world):
            lo, hi = online_slice(start, m, r, world)
            ra, rw = np.zeros((C, D)), np.zeros(C)
            for i in range(lo, hi):
                pops = (cv != dense[i].astype(np.uint8)[None, :]).sum(axis=1)
                pred = int(np.argmin(pops))
                dt = pops[y[i]] / D
                ra[y[i]] = ra[y[i]] + dense[i] * dt
                rw[y[i]] += dt
                if pred != y[i]:
                    ra[pred] = ra[pred] + dense[i] * (-gamma * (1.0 - pops[pred] / D))
            d_acc += ra
            d_w += rw
        acc = acc + d_acc
        weight = weight + d_w
        cv = binarize(acc, weight)
    return acc, weight, cv


@pytest.mark.parametrize("world", [2, 4])
def test_online_delta_mode_is_within_tolerance_of_exact(world):
    """North-star contract for sharded online training: accumulators within
    1e-5 relative of the exact reference semantics, identical class HVs."""
    rng = np.random.default_rng(5)
    C, D, n, bsz = 3, 256, 240, 32
    centers = rng.integers(0, 2, (C, D), dtype=np.uint8)
    y = (np.arange(n) % C).astype(np.int32)
    flip = rng.random((n, D)) < 0.2
    enc = O.pack_rows(centers[y] ^ flip.astype(np.uint8))
    tb = O.generate_random(1, D, 11)
    exact = O.NaiveModel(C, D, tb).train_online(enc, y, bsz)
    acc, weight, cv = _online_delta_reference(enc, y, C, D, bsz, 1.0, world, tb)
    np.testing.assert_allclose(acc, exact.acc, rtol=1e-5, atol=1e-9)
    np.testing.assert_allclose(weight, exact.weight, rtol=1e-5)
    np.testing.assert_array_equal(cv, exact.cv)


def test_word_slices_partition_rows():
    from paper_2206_04746_b200.device import word_slice
    for words in (1, 7, 32, 313, 1024):
        for world in (1, 2, 3, 4, 8):
            if world > words:
                continue
            sl = [word_slice(words, r, world) for r in range(world)]
            assert sl[0][0] == 0 and sum(n for _, n in sl) == words
            assert all(a[0] + a[1] == b[0] for a, b in zip(sl, sl[1:]))
            assert max(n for _, n in sl) - min(n for _, n in sl) <= 1


def _dsliced_worker(rank, world, port, enc, y, C, D, bsz, gamma, tb, q):
    """NumPy restatement of device.DSlicedOnline on one rank: partial popcounts
    over its words, gloo all-reduce, sample-ordered updates of its columns."""
    from paper_2206_04746_b200.device import word_slice
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    W = enc.shape[1]
    w0, nw = word_slice(W, rank, world)
    j0, j1 = 32 * w0, min(D, 32 * (w0 + nw))
    dense = O.unpack_rows(enc, D)[:, j0:j1]
    tbits = O.unpack_rows(tb, D)[0, j0:j1]
    n = enc.shape[0]
    first = min(bsz, n)
    acc = np.zeros((C, j1 - j0))
    weight = np.zeros(C)
    counts = np.zeros(C, np.int64)
    for c in range(C):
        acc[c] = dense[:first][y[:first] == c].sum(axis=0)
        weight[c] = counts[c] = (y[:first] == c).sum()

    def binarize():
        tw = 2.0 * acc
        return np.where(tw > weight[:, None], 1, np.where(tw < weight[:, None], 0, tbits[None, :])).astype(np.uint8)

    cv = binarize()
    for start in range(0, n, bsz):
        m = min(bsz, n - start)
        part = np.stack([(cv != dense[i][None, :]).sum(axis=1) for i in range(start, start + m)]).astype(np.int32)
        pt = torch.from_numpy(part)
        dist.all_reduce(pt)
        pops = pt.numpy()
        for k, i in enumerate(range(start, start + m)):
            pred = int(np.argmin(pops[k]))
            t = int(y[i])
            dt = pops[k][t] / D
            acc[t] = np.where(dense[i] == 1, acc[t] + dt, acc[t])
            weight[t] += dt
            counts[t] += 1
            if pred != t:
                pen = -gamma * (1.0 - pops[k][pred] / D)
                acc[pred] = np.where(dense[i] == 1, acc[pred] + pen, acc[pred])
        cv = binarize()
    parts = [None] * world
    dist.all_gather_object(parts, (acc, cv, weight, counts))
    if rank == 0:
        q.put(parts)
    dist.destroy_process_group()


@pytest.mark.parametrize("world,D", [(2, 256), (3, 1000)])
def test_dsliced_online_is_bit_exact_with_one_process(world, D):
    """The D-sliced multi-GPU online protocol (one all-reduce of integer
    popcounts per batch) reproduces the exact reference trainer bit for bit."""
    rng = np.random.default_rng(world + D)
    C, n, bsz = 3, 150, 32
    centers = rng.integers(0, 2, (C, D), dtype=np.uint8)
    y = (np.arange(n) % C).astype(np.int32)
    enc = O.pack_rows(centers[y] ^ (rng.random((n, D)) < 0.25).astype(np.uint8))
    tb = O.generate_random(1, D, 13)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_dsliced_worker, args=(r, world, port, enc, y, C, D, bsz, 1.0, tb, q))
             for r in range(world)]
    for p in procs:
        p.start()
    parts = q.get(timeout=180)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    acc = np.concatenate([a for a, _, _, _ in parts], axis=1)
    cv = np.concatenate([c for _, c, _, _ in parts], axis=1)
    exact = O.NaiveModel(C, D, tb).train_online(enc, y, bsz)
    np.testing.assert_array_equal(acc, exact.acc)
    np.testing.assert_array_equal(cv, exact.cv)
    for _, _, w, cnt in parts:
        np.testing.assert_array_equal(w, exact.weight)
        np.testing.assert_array_equal(cnt, exact.counts.astype(np.int64))
