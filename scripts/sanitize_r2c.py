"""Small-shape driver of the late round-2 two-class online changes for
compute-sanitizer (memcheck / racecheck / synccheck): one CTA per SM with the
items past the item CTAs drawn from a per-batch counter, class-weight tasks
that skip 32-row groups without true samples, and staging that issues raw
loads two chunks ahead (csrc/hv_online.cu replay_merged_mw). The result is
checked against the 160-CTA static schedule (HVB200_ONLINE_DYNAMIC=0).

usage: compute-sanitizer --tool memcheck python scripts/sanitize_r2c.py
"""
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2206_04746_b200 import device as dv  # noqa: E402


def main():
    cbk = dv.DeviceCodebook.make(64, 16, 10000, seed=5)
    eng = dv.Engine(cbk, 2)
    b8, _ = eng.synth(0, 3 * 1024 + 300, 1, 7)
    enc = eng.encode(b8)
    rng = np.random.default_rng(3)
    y = torch.from_numpy((rng.random(enc.shape[0]) < 0.05).astype(np.int32)).to(enc.device)
    res = []
    for dyn in ("1", "0"):
        os.environ["HVB200_ONLINE_DYNAMIC"] = dyn
        res.append(tuple(t.clone() for t in eng.train_online(enc, y, 1024, 0.5)))
    del os.environ["HVB200_ONLINE_DYNAMIC"]
    for a, b in zip(res[0], res[1]):
        assert torch.equal(a, b)
    eng.dc.check()
    torch.cuda.synchronize()
    print("sanitize_r2c: dynamic and static schedules ran and agreed")


if __name__ == "__main__":
    main()
