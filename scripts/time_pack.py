"""Drives hv_pack / hv_unpack on a large matrix for an ncu launch list
(kernel durations -> GB/s of dense bytes + packed bytes moved).

usage: ncu --metrics gpu__time_duration.sum --csv ... python scripts/time_pack.py ROWS DIM
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2206_04746_b200 import hypervec as hv  # noqa: E402

rows, dim = int(sys.argv[1]), int(sys.argv[2])
dense = (np.random.default_rng(0).random((rows, dim)) < 0.5).astype(np.uint8)
for _ in range(2):
    p = hv.pack(hv.DenseBitMatrix(rows, dim, dense))
    u = hv.unpack(p)
assert np.array_equal(u.bits, dense)
print(f"pack/unpack {rows} x {dim}: dense {rows * dim / 1e9:.3f} GB, packed {p.words.nbytes / 1e9:.3f} GB")
