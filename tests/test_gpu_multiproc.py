"""Multi-process tests of the engine's N > 1 paths on the one GPU of a test
box (ranks share it; gloo for the torch.distributed plumbing, CUDA IPC for the
fused peer-memory collectives):

* `bench.py` under torchrun with 2 ranks (HVB200_BENCH_SHARE_GPU=1): the
  timed step's class vectors and predicted labels are identical to the N = 1
  run, and so are the word-sliced online trainer's accumulators and class
  vectors (stitched from both ranks);
* 2 processes driving device.DSlicedOnline (popcount all-reduce through
  torch.distributed, and fused over peer memory) and the delta-mode
  Engine.train_online_sharded against the C oracle: word-sliced bit-exact,
  delta mode within 1e-5 relative with class vectors equal away from exact
  ties (model.cpp:250-301, experiment.cpp:148-178).
"""
import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

import oracle_ref as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
ROOT = Path(__file__).resolve().parents[1]


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _bench(tmp, world, rows):
    env = dict(os.environ, HVB200_BENCH_SHARE_GPU="1")
    args = ["bench.py", "--gpus", str(world), "--rows", str(rows), "--steps", "2", "--warmup", "3", "--no-e2e",
            "--no-cpu", "--online-batch", "1024", "--dump", str(tmp)]
    if world > 1:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
               "--master-addr", "127.0.0.1", "--master-port", str(_port()), *args]
    else:
        cmd = [sys.executable, *args]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    return r.stdout


def _stitch(tmp, world, name):
    parts = []
    for r in range(world):
        w0, nw = np.load(tmp / f"online_w0_{r}.npy")
        a = np.load(tmp / f"online_{name}_{r}.npy")
        parts.append((w0, a))
    return np.concatenate([a for _, a in sorted(parts, key=lambda t: t[0])], axis=1)


def test_bench_two_ranks_equal_one_rank(tmp_path):
    rows = 200_000
    one, two = tmp_path / "n1", tmp_path / "n2"
    _bench(one, 1, rows)
    out = _bench(two, 2, rows)
    assert '"n_gpus": 2' in out
    np.testing.assert_array_equal(np.load(one / "cv.npy"), np.load(two / "cv.npy"))
    p1 = np.load(one / "pred_0.npy")
    p2 = np.concatenate([np.load(two / f"pred_{r}.npy") for r in sorted(range(2), key=lambda r: int(
        np.load(two / f"pred_lo_{r}.npy")[0]))])
    np.testing.assert_array_equal(p1, p2)
    # online: word-sliced exact (2 ranks) == single-GPU exact trainer, bit for bit
    cv1, acc1 = np.load(one / "online_cv_0.npy"), np.load(one / "online_acc_0.npy")
    np.testing.assert_array_equal(_stitch(two, 2, "cv"), cv1)
    np.testing.assert_array_equal(_stitch(two, 2, "acc").view(np.uint64), acc1.view(np.uint64))


def test_two_process_online_modes_vs_oracle(tmp_path):
    import torch.multiprocessing as mp

    sys.path.insert(0, str(Path(__file__).resolve().parent))
    import mp_workers

    F, C, D, rows, bsz, world = 561, 6, 10000, 6000, 1000, 2
    mp.spawn(mp_workers.online_ranks, args=(world, _port(), str(tmp_path), F, C, D, rows, bsz, 13, 3),
             nprocs=world, join=True)
    inp = np.load(tmp_path / "inputs.npz")
    enc, labels, tb = inp["enc"].view(np.uint32), inp["labels"], inp["tiebreak"].view(np.uint32)
    om = O.NaiveModel(C, D, tb).train_online(enc, labels, bsz)
    sl = [np.load(tmp_path / f"sliced_{r}.npz") for r in range(world)]
    sl.sort(key=lambda z: int(z["w0"]))
    acc = np.concatenate([z["acc"] for z in sl], axis=1)
    cv = np.concatenate([z["cv"] for z in sl], axis=1).view(np.uint32)
    np.testing.assert_array_equal(acc.view(np.uint64), om.acc.view(np.uint64))
    np.testing.assert_array_equal(cv, om.class_vectors)
    for z in sl:
        np.testing.assert_array_equal(z["weight"].view(np.uint64), om.weight.view(np.uint64))
        np.testing.assert_array_equal(z["counts"].astype(np.uint64), om.counts.astype(np.uint64))
    order = np.argsort([int(np.load(tmp_path / f"sliced_{r}.npz")["w0"]) for r in range(world)])
    pe = [np.load(tmp_path / f"peer_{r}.npz") for r in order]
    acc_p = np.concatenate([z["acc"] for z in pe], axis=1)
    np.testing.assert_array_equal(np.concatenate([z["cv"] for z in pe], axis=1).view(np.uint32), om.class_vectors)
    np.testing.assert_array_equal(acc_p.view(np.uint64), om.acc.view(np.uint64))
    # delta mode: replicated result on every rank, within 1e-5 of the exact trainer
    for r in range(world):
        d = np.load(tmp_path / f"delta_{r}.npz")
        rel = np.abs(d["acc"] - om.acc) / np.maximum(np.abs(om.acc), 1.0)
        assert rel.max() <= 1e-5, rel.max()
        np.testing.assert_array_equal(d["counts"].astype(np.uint64), om.counts.astype(np.uint64))
        diff = O.unpack_rows((d["cv"].view(np.uint32) ^ om.class_vectors), D).astype(bool)
        margin = np.abs(2.0 * om.acc - om.weight[:, None])
        assert np.all(margin[diff] <= 1e-9 * np.repeat(om.weight[:, None], D, 1)[diff]), "class bit flip away from a tie"
