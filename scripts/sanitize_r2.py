"""Small-shape driver of the round-2 kernels for compute-sanitizer
(memcheck / racecheck): TMA-staged class counts on pitched rows with class
segments inside staged batches, the pitched and two-class predict scans,
pack/unpack on the three paths, the 32-bin table encoder and the device
single-pair helpers. Each result is also checked against a second path.

usage: compute-sanitizer --tool memcheck python scripts/sanitize_r2.py
"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2206_04746_b200 import device as dv  # noqa: E402
from paper_2206_04746_b200 import hypervec as hv  # noqa: E402


def main():
    for D, C, rows in ((1000, 3, 5000), (96, 2, 2100), (20000, 5, 700)):
        cbk = dv.DeviceCodebook.make(24, 16, D, seed=D)
        eng = dv.Engine(cbk, C)
        bins8, _ = eng.synth(0, rows, 0, 3)
        labels = torch.randint(0, C, (rows,), dtype=torch.int32, device="cuda")
        flat = eng.encode(bins8)
        pit = eng.encode(bins8, pitched=True)
        c1, r1 = eng.zero_counts()
        c2, r2 = eng.zero_counts()
        eng.class_counts(flat, labels, c1, r1)
        eng.class_counts(pit, labels, c2, r2)
        assert torch.equal(c1, c2) and torch.equal(r1, r2)
        cv = eng.binarize(c1, r1)
        assert torch.equal(eng.predict(cv, flat), eng.predict(cv, pit))
        pops = torch.empty((rows, C), dtype=torch.int32, device="cuda")
        assert torch.equal(eng.predict(cv, pit, popcounts=pops), eng.predict(cv, flat))
    for D in (10000, 1000, 999):
        dense = (np.random.default_rng(D).random((300, D)) < 0.5).astype(np.uint8)
        p = hv.pack(hv.DenseBitMatrix(300, D, dense))
        assert np.array_equal(hv.unpack(p).bits, dense)
    cbk = dv.DeviceCodebook.make(342, 32, 10000, seed=1)
    eng = dv.Engine(cbk, 2)
    bins = torch.randint(0, 32, (600, dv.bins_pitch(342)), dtype=torch.uint8, device="cuda")
    eng.encode(bins)
    a = np.arange(313, dtype=np.uint32)
    hv.hamming_distance_words(a, a[::-1].copy(), 10000)
    hv.cosine_similarity(np.linspace(-1, 1, 64), np.array([5, 7], np.uint32), 64)
    eng.dc.check()
    torch.cuda.synchronize()
    print("sanitize_r2: all paths ran and agreed")


if __name__ == "__main__":
    main()
