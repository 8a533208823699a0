"""Online trainer per-batch phase times at each BASELINE shape on a sample of
rows (batch 256 / 1,024 / 8,192). Run with HVB200_ONLINE_PROFILE=1 for the
per-phase split (CTA 0's view, each phase including its grid barrier).

usage: HVB200_ONLINE_PROFILE=1 python scripts/online_phases.py H I L E M M20 > profiles/online_phases_r2.txt
"""
import os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_2206_04746_b200 import device as dv
cfgs = {"H": (561, 6, 10000, 200_000, 0), "I": (617, 26, 10000, 100_000, 0), "L": (617, 100, 32768, 60_000, 0), "E": (342, 2, 10000, 200_000, 1), "M": (784, 10, 10000, 100_000, 0), "M20": (784, 10, 20000, 60_000, 0),
        "M8k": (784, 10, 8192, 100_000, 0), "M16k": (784, 10, 16384, 60_000, 0)}
for name in sys.argv[1:]:
    F, C, D, rows, lk = cfgs[name]
    cbk = dv.DeviceCodebook.make(F, 16, D, seed=3)
    eng = dv.Engine(cbk, C)
    b8, y = eng.synth(0, rows, lk, 7)
    enc = eng.encode(b8)
    for bs in (256, 1024, 8192):
        eng.train_online(enc, y, bs); torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); eng.train_online(enc, y, bs); e.record(); torch.cuda.synchronize()
        print(f"{name} C={C} D={D} rows={rows} batch {bs}: {s.elapsed_time(e):.3f} ms, {s.elapsed_time(e)*1e3/((rows+bs-1)//bs):.2f} us/batch", flush=True)
