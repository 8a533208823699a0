"""Small-batch online training: persistent cooperative kernel vs the cluster trainer
(UCI-HAR shape, batch 1..64); prints one JSON line per batch size. GPU only."""
import os, sys, json, torch
sys.path.insert(0, os.getcwd())
from paper_2206_04746_b200 import device as dv
F, B, D, C, rows = 561, 16, 10000, 6, 8000
cbk = dv.DeviceCodebook.make(F, B, D, seed=3)
eng = dv.Engine(cbk, C)
bins8, labels = eng.synth(0, rows, 0, 7)
enc = eng.encode(bins8)
torch.cuda.synchronize()
for bs in (1, 2, 4, 8, 12, 16, 24, 32, 48, 64):
    out = {}
    for mode in ("0", "64"):
        os.environ["HVB200_ONLINE_CLUSTER"] = mode
        eng.train_online(enc, labels, bs)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        r = eng.train_online(enc, labels, bs)
        e.record(); torch.cuda.synchronize()
        out[mode] = (s.elapsed_time(e), r)
    same = all(torch.equal(a, b) for a, b in zip(out["0"][1], out["64"][1]))
    print(json.dumps({"batch": bs, "persistent_ms": round(out["0"][0], 3), "cluster_ms": round(out["64"][0], 3), "identical": same}))
