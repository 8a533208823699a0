"""A/B of the online weight chains: inside the items / list phase (HVB200_ONLINE_WTASK=0) vs
separate tasks on spare CTAs (default), several BASELINE shapes. GPU only."""
import os, sys, torch, json
sys.path.insert(0, os.getcwd())
from paper_2206_04746_b200 import device as dv
cases = [("H", 561, 6, 10000, 800_000, 256, 0), ("H", 561, 6, 10000, 800_000, 1024, 0), ("H", 561, 6, 10000, 800_000, 8192, 0),
         ("M", 784, 10, 10000, 56_000, 1024, 0), ("M", 784, 10, 1024, 56_000, 1024, 0), ("E", 342, 2, 10000, 524_288, 1024, 1),
         ("H32", 561, 6, 10000, 8000, 32, 0)]
for tag, F, C, D, rows, bs, lk in cases:
    cbk = dv.DeviceCodebook.make(F, 16, D, seed=1)
    eng = dv.Engine(cbk, C)
    bins8, labels = eng.synth(0, rows, lk, 7)
    enc = eng.encode(bins8)
    res = {}
    for mode in ("0", "1", "0", "1"):
        os.environ["HVB200_ONLINE_WTASK"] = mode
        eng.train_online(enc, labels, bs); torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); r = eng.train_online(enc, labels, bs); e.record(); torch.cuda.synchronize()
        res.setdefault(mode, []).append(round(s.elapsed_time(e), 3))
    print(json.dumps({"case": tag, "D": D, "batch": bs, "in_item_ms": res["0"], "task_ms": res["1"]}))
    del eng, bins8, enc
