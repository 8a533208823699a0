"""CHB-MIT-shaped online training on a 262,144-row prefix (256 batches of 1,024):
a short run of the persistent online kernel for ncu captures. GPU only."""
import os
import sys

import torch

sys.path.insert(0, os.getcwd())
from paper_2206_04746_b200 import device as dv  # noqa: E402

F, B, D, C, rows = 342, 16, 10000, 2, 262_144
cbk = dv.DeviceCodebook.make(F, B, D, seed=3)
eng = dv.Engine(cbk, C)
bins8, labels = eng.synth(0, rows, 1, 7)
enc = eng.encode(bins8)
eng.train_online(enc, labels, 1024)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
eng.train_online(enc, labels, 1024)
e.record()
torch.cuda.synchronize()
print(f"online {rows} rows batch 1024: {s.elapsed_time(e):.3f} ms ({s.elapsed_time(e) * 1e3 / (rows / 1024):.2f} us/batch)")
