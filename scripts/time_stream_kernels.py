"""Times the HBM-streaming kernels — classical column counts and the
few-class Hamming scan — with CUDA events at the BASELINE shapes, against the
measured HBM peak (MEASURED_PEAKS.json). Algorithmic bytes: counts read 4W
bytes per train row (+ the 4-byte label and permutation entry); predict reads
4W bytes per row and writes a 4-byte label.

usage: python scripts/time_stream_kernels.py > profiles/stream_kernels_<round>.jsonl
"""
import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2206_04746_b200 import device as dv  # noqa: E402

SHAPES = [  # name, F, C, D, rows (all rows encoded; 80 % train / 20 % predict)
    ("E", 342, 2, 10000, 7_060_000),
    ("H", 561, 6, 10000, 2_000_000),
    ("I", 617, 26, 10000, 1_000_000),
    ("M1k", 784, 10, 1024, 8_000_000),
    ("M20k", 784, 10, 20000, 1_000_000),
]


def timed(fn, reps=10):
    st = torch.cuda.current_stream()
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        fn()
        b.record(st)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


def main():
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    peak = peaks.get("hbm_gbs", 6650.0)
    only = set(sys.argv[1:])
    for name, F, C, D, rows in SHAPES:
        if only and name not in only:
            continue
        cbk = dv.DeviceCodebook.make(F, 16, D, seed=1)
        eng = dv.Engine(cbk, C)
        bins8, labels = eng.synth(0, rows, 1 if name == "E" else 0, 7)
        enc = eng.encode(bins8, pitched=True)  # the engine's resident layout (16-byte rows)
        del bins8
        W = enc.shape[1]
        ntr = rows * 4 // 5
        counts, crow = eng.zero_counts()
        cv, _, _ = eng.train_classical(enc[:ntr], labels[:ntr])
        pred = torch.empty(rows - ntr, dtype=torch.int32, device=enc.device)

        def count():
            counts.zero_()
            crow.zero_()
            eng.class_counts(enc[:ntr], labels[:ntr], counts, crow)

        tc = timed(count)
        tp = timed(lambda: eng.predict(cv, enc[ntr:], labels=pred))
        bc = ntr * (4 * W + 8)
        bp = (rows - ntr) * (4 * W + 4)
        for stage, ms, nb, n in (("class_counts", tc, bc, ntr), ("predict", tp, bp, rows - ntr)):
            gbs = nb / (ms / 1e3) / 1e9
            print(json.dumps({"shape": name, "F": F, "C": C, "D": D, "rows": n, "stage": stage, "ms": round(ms, 4),
                              "alg_bytes": nb, "gb_s": round(gbs, 1), "hbm_peak_gb_s": peak,
                              "frac": round(gbs / peak, 4)}), flush=True)
        del enc


if __name__ == "__main__":
    main()
