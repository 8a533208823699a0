"""Online training per-batch time for small batches (1 / 4 / 16 / 32 rows) at the
UCI-HAR shape: the cluster trainer (<= 16 rows) and the persistent kernel.

usage: python scripts/online_small_batches.py
"""
import os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_2206_04746_b200 import device as dv
cbk = dv.DeviceCodebook.make(561, 16, 10000, seed=3)
eng = dv.Engine(cbk, 6)
b8, y = eng.synth(0, 10000, 0, 7)
enc = eng.encode(b8)
for bs in (1, 4, 16, 32):
    eng.train_online(enc, y, bs); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); eng.train_online(enc, y, bs); e.record(); torch.cuda.synchronize()
    print(f"H 10k rows batch {bs}: {s.elapsed_time(e):.3f} ms, {s.elapsed_time(e)*1e3/((10000+bs-1)//bs):.3f} us/batch", flush=True)
