"""Small driver for ncu captures of individual kernels at a named shape.

usage: python scripts/probe_kernels.py predict|online|classical F C D ROWS [BATCH]
"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2206_04746_b200 import device as dv  # noqa: E402


def main():
    what, F, C, D, rows = sys.argv[1], *map(int, sys.argv[2:6])
    bsz = int(sys.argv[6]) if len(sys.argv) > 6 else 1024
    cbk = dv.DeviceCodebook.make(F, 16, D, seed=1)
    eng = dv.Engine(cbk, C)
    bins8, labels = eng.synth(0, rows, 0, 7)
    enc = eng.encode(bins8)
    cv, _, _ = eng.train_classical(enc, labels)
    torch.cuda.synchronize()
    if what == "predict":
        eng.predict(cv, enc)
    elif what == "online":
        eng.train_online(enc, labels, bsz)
    elif what == "classical":
        eng.train_classical(enc, labels)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
