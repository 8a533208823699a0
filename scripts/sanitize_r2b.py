"""Small-shape driver of the late round-2 paths for compute-sanitizer
(memcheck / racecheck / synccheck): the streamed fold staging (one encoder
launch waiting on the rows the copy stream lands, hv_stage.cu) against the
chunked pipeline, including a bad bin that aborts the launch; the 12-warp
table encoder against the generic kernel; and the two-class online trainer's
narrow replay items (replay_merged_mw) against the 8-word items.

usage: compute-sanitizer --tool memcheck python scripts/sanitize_r2b.py
"""
import ctypes as C
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2206_04746_b200 import _native as N  # noqa: E402
from paper_2206_04746_b200 import device as dv  # noqa: E402
from paper_2206_04746_b200 import hypervec as hv  # noqa: E402


def fold(bins, y, ntr, F, B, D, cb, etb, mtb, env):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        L = N.lib()
        ctx = N.context(0)
        f = C.c_void_p()
        p = lambda a: C.c_void_p(a.ctypes.data)
        N.check(L.hv_fold_encode_train(ctx.handle, p(bins), ntr, p(y), C.c_void_p(bins.ctypes.data + ntr * F * 4),
                                       bins.shape[0] - ntr, F, p(cb.id_vectors.words), p(cb.value_vectors.words), B, D,
                                       p(etb), 2, C.byref(f)))
        out = np.zeros(bins.shape[0] - ntr, np.int32)
        N.check(L.hv_fold_predict(ctx.handle, f, p(mtb), p(out)))
        L.hv_fold_destroy(f)
        return out
    finally:
        for k, v in old.items():
            os.environ.pop(k, None)
            if v is not None:
                os.environ[k] = v


def main():
    rng = np.random.default_rng(5)
    F, B, D, rows, ntr = 342, 16, 2000, 6000, 4800
    cb = hv.make_codebook(hv.GenerationStrategy.kRandom, hv.BindingStrategy.kIdLevel, F, B, D, 11)
    etb = np.ascontiguousarray(hv.generate_random(1, D, 12).words)
    mtb = np.ascontiguousarray(hv.generate_random(1, D, 13).words)
    bins = rng.integers(0, B, (rows, F)).astype(np.uint32)
    y = (rng.random(ntr) < 0.3).astype(np.int32)
    a = fold(bins, y, ntr, F, B, D, cb, etb, mtb, {"HVB200_STAGE_MB": "1"})
    b = fold(bins, y, ntr, F, B, D, cb, etb, mtb, {"HVB200_STAGE_STREAM": "0", "HVB200_STAGE_MB": "1"})
    assert np.array_equal(a, b)
    bad = bins.copy()
    bad[3000, 7] = 16
    try:
        fold(bad, y, ntr, F, B, D, cb, etb, mtb, {"HVB200_STAGE_MB": "1"})
        raise AssertionError("bad bin accepted")
    except Exception as e:  # noqa: BLE001
        assert "bin index 16" in str(e), e
    # 12-warp table encoder vs the generic kernel
    cbk = dv.DeviceCodebook.make(342, 16, 10000, seed=3)
    eng = dv.Engine(cbk, 2)
    b8, lab = eng.synth(0, 3000, 1, 7)
    fast = eng.encode(b8)
    os.environ["HVB200_ENCODE_GENERIC"] = "1"
    gen = eng.encode(b8)
    del os.environ["HVB200_ENCODE_GENERIC"]
    assert torch.equal(fast, gen)
    # two-class online trainer: 4-word replay items vs 8-word items
    res = []
    for mw in ("4", "8"):
        os.environ["HVB200_ONLINE_MW"] = mw
        res.append(tuple(t.clone() for t in eng.train_online(fast, lab, 256, 0.5)))
    del os.environ["HVB200_ONLINE_MW"]
    for x, z in zip(res[0], res[1]):
        assert torch.equal(x, z)
    eng.dc.check()
    torch.cuda.synchronize()
    print("sanitize_r2b: all paths ran and agreed")


if __name__ == "__main__":
    main()
