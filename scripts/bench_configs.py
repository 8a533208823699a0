"""Per-configuration stage benchmark: every BASELINE.json config
on one B200, each stage timed with CUDA events on the launching stream, next
to the reference library (oracle/_ref/ref_bench) on a bounded sample of the
same synthetic workload on all host cores.

usage: python scripts/bench_configs.py [--only I,H,M,E,L] [--no-cpu] > profiles/configs_rNN.jsonl

Configs (BASELINE.json `configs`, SURVEY.md §8 shorthand):
  I  ISOLET-shaped   F=617 C=26  D=10000, classical, N=1M (steady state)
  H  UCI-HAR-shaped  F=561 C=6   D=10000, online, batch sweep 1..8192
  M  MNIST-shaped    F=784 C=10  D sweep 1k..20k, classical + online(1024)
  E  CHB-MIT-shaped  F=342 C=2   D=10000, N=7.06M, online(1024) (classical is bench.py)
  L  Large           F=617 C=100 D=32768, N=10M, classical vs online(1024)
Inputs are resident in HBM; bins (uint8) + hypervectors exceed L2 for every
N >= 1M line. One line per (config, trainer, D, batch).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
REF_BENCH = ROOT / "oracle" / "_ref" / "ref_bench"

from paper_2206_04746_b200 import device as dv  # noqa: E402

PEAKS = {}
try:
    PEAKS = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
except Exception:
    pass
HBM = PEAKS.get("hbm_gbs", 6450.0)


def split(rows):
    train = min(rows - 1, max(1, rows * 4 // 5))
    return train, rows - train


def timed(fn, reps=1):
    """Median of `reps` individually timed calls after two warm-up calls (the
    first call of a path pays lazy module loading and memory-pool growth)."""
    s = torch.cuda.current_stream()
    fn()
    fn()
    torch.cuda.synchronize()
    times = []
    for _ in range(max(reps, 1)):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        out = fn()
        e1.record(s)
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    return sorted(times)[len(times) // 2], out


def ref_cpu(F, C, D, rows, trainer, batch, label_kind, target_s=8.0):
    if not REF_BENCH.exists():
        return None
    threads = os.cpu_count() or 1

    def run(n):
        cmd = [str(REF_BENCH), "--features", str(F), "--classes", str(C), "--dim", str(D), "--rows", str(n),
               "--bins", "16", "--threads", str(threads), "--labels", "chbmit" if label_kind == 1 else "mod",
               "--trainer", trainer, "--batch", str(batch), "--seed", "1", "--data-seed", "7"]
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
        if r.returncode != 0:
            raise RuntimeError(r.stderr)
        return json.loads(r.stdout.strip().splitlines()[-1])

    cal = run(1024)
    n = int(min(rows, max(1024, 1024 * target_s / max(cal["total_s"], 1e-3))))
    r = run(n)
    return {"dp_per_s": round(r["dp_per_s"], 1), "rows": n, "threads": threads, "total_s": r["total_s"],
            "encode_s": r["encode_s"], "train_s": r["train_s"], "predict_s": r["predict_s"]}


def one(tag, F, C, D, rows, trainer, batch, label_kind=0, cpu=True, reps=3):
    W = (D + 31) // 32
    ntr, nte = split(rows)
    cbk = dv.DeviceCodebook.make(F, 16, D, seed=1)
    eng = dv.Engine(cbk, C)
    eng.dc.bind()
    bins8, labels = eng.synth(0, rows, label_kind, 7)
    # classical with < 32 classes keeps the engine's pitched rows (16-byte rows:
    # TMA-staged counts, uint4 predict); the online trainer reads unpitched rows
    pitched = trainer == "classical" and C < 32
    enc = eng.pitched_empty(rows) if pitched else torch.empty((rows, W), dtype=torch.int32, device=eng.dev)
    ms_enc, _ = timed(lambda: eng.encode(bins8, out=enc), reps)
    yt = labels[:ntr]
    if trainer == "classical":
        ms_train, (cv, _, _) = timed(lambda: eng.train_classical(enc[:ntr], yt), reps)
    else:
        r = 1 if batch < 64 else reps
        ms_train, res = timed(lambda: eng.train_online(enc[:ntr], yt, batch), r)
        cv = res[3]
    pred = torch.empty(nte, dtype=torch.int32, device=eng.dev)
    ms_pred, _ = timed(lambda: eng.predict(cv, enc[ntr:], labels=pred), reps)
    eng.dc.check()
    total = ms_enc + ms_train + ms_pred
    acc = (pred == labels[ntr:]).float().mean().item() if nte else None
    f_sm = PEAKS.get("sm_max_mhz", 1965.0) * 1e6
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    line = {
        "config": tag, "features": F, "classes": C, "dim": D, "rows": rows, "train_rows": ntr, "test_rows": nte,
        "trainer": trainer, "batch_size": batch if trainer == "online" else None, "pitched_rows": pitched,
        "dp_per_s": round(rows / (total / 1e3), 1),
        "ms": {"encode": round(ms_enc, 3), "train": round(ms_train, 3), "predict": round(ms_pred, 3)},
        "encode": {"dp_per_s": round(rows / (ms_enc / 1e3), 1),
                   "bound_words_per_s": round(rows * F * W / (ms_enc / 1e3) / 1e9, 1),
                   "ceiling_frac": round(rows * F * W / (ms_enc / 1e3) / (sms * 32 * f_sm), 4),
                   "hbm_frac": round(rows * (F + 4 * W) / (ms_enc / 1e3) / 1e9 / HBM, 5)},
        "train": {"dp_per_s": round(ntr / (ms_train / 1e3), 1),
                  "hbm_gbs": round(ntr * (4 * W + 4) / (ms_train / 1e3) / 1e9, 1),
                  "hbm_frac": round(ntr * (4 * W + 4) / (ms_train / 1e3) / 1e9 / HBM, 4)},
        "predict": {"dp_per_s": round(nte / (ms_pred / 1e3), 1) if nte else None,
                    "hbm_gbs": round(nte * (4 * W + 4) / (ms_pred / 1e3) / 1e9, 1),
                    "hbm_frac": round(nte * (4 * W + 4) / (ms_pred / 1e3) / 1e9 / HBM, 4),
                    "popc_per_s_T": round(nte * C * W / (ms_pred / 1e3) / 1e12, 3)},
        "test_accuracy": round(acc, 4) if acc is not None else None,
    }
    if cpu:
        ref = ref_cpu(F, C, D, rows, trainer, batch, label_kind)
        line["cpu_reference"] = ref
        if ref:
            line["speedup_vs_cpu"] = round(line["dp_per_s"] / ref["dp_per_s"], 1)
    print(json.dumps(line), flush=True)
    del bins8, labels, enc, eng
    torch.cuda.empty_cache()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="I,H,M,E,L")
    ap.add_argument("--no-cpu", action="store_true")
    a = ap.parse_args()
    only = set(a.only.split(","))
    cpu = not a.no_cpu
    torch.cuda.set_device(0)
    if "I" in only:
        one("I", 617, 26, 10000, 1_000_000, "classical", 0, cpu=cpu)
    if "H" in only:
        for b in (1, 32, 256, 1024, 8192):
            one("H", 561, 6, 10000, 10_000, "online", b, cpu=cpu)
        for b in (256, 1024, 8192):
            one("H", 561, 6, 10000, 1_000_000, "online", b, cpu=cpu)
    if "M" in only:
        for d in (1024, 2048, 4096, 8192, 10000, 16384, 20000):
            one("M", 784, 10, d, 70_000, "classical", 0, cpu=cpu)
            one("M", 784, 10, d, 70_000, "online", 1024, cpu=cpu)
        one("M", 784, 10, 10000, 1_000_000, "classical", 0, cpu=cpu)
    if "E" in only:
        one("E", 342, 2, 10000, 7_060_000, "online", 1024, label_kind=1, cpu=cpu)
    if "L" in only:
        one("L", 617, 100, 32768, 10_000_000, "classical", 0, cpu=cpu, reps=1)
        one("L", 617, 100, 32768, 10_000_000, "online", 1024, cpu=cpu, reps=1)


if __name__ == "__main__":
    main()
