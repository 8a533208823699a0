"""Breaks the bench's e2e leg (hv_fold_encode_train + hv_fold_predict from
pinned host uint32 bins) into its parts on the CHB-MIT workload: host
narrowing alone (hv_host_narrow_bins over all rows), each fold call, and the
device-resident encode of the same rows, so the gap between `e2e` and `value`
can be attributed. Run with HVB200_STAGE_PROFILE=1 for the per-call
slot-wait / narrow split.

usage: python scripts/probe_e2e.py [rows]
"""
import ctypes as C
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2206_04746_b200 import _native as N  # noqa: E402
from paper_2206_04746_b200 import device as dv  # noqa: E402


def main():
    rows = int(sys.argv[1]) if len(sys.argv) > 1 else 7_060_000
    F, B, D, Cc = 342, 16, 10000, 2
    n_tr = rows * 4 // 5
    n_te = rows - n_tr
    print(f"nproc {os.cpu_count()} rows {rows} HOST_THREADS={os.environ.get('HVB200_HOST_THREADS')} "
          f"STAGE_MB={os.environ.get('HVB200_STAGE_MB')}", flush=True)
    cbk = dv.DeviceCodebook.make(F, B, D, seed=1)
    eng = dv.Engine(cbk, Cc)
    b8, y = eng.synth(0, rows, 1, 7)
    b32 = torch.empty((rows, F), dtype=torch.int32, pin_memory=True)
    b32.copy_(b8[:, :F].to(torch.int32).cpu())
    lab = torch.empty(n_tr, dtype=torch.int32, pin_memory=True)
    lab.copy_(y[:n_tr].cpu())
    del b8, y
    L = N.lib()
    ldb = dv.bins_pitch(F)
    out8 = torch.empty((rows, ldb), dtype=torch.uint8, pin_memory=True)
    bad = C.c_uint64()
    for rep in range(3):
        t = time.perf_counter()
        N.check(L.hv_host_narrow_bins(C.c_void_p(b32.data_ptr()), rows, F, B, C.c_void_p(out8.data_ptr()), ldb,
                                      C.byref(bad)))
        dt = time.perf_counter() - t
        print(f"host narrow all rows: {dt * 1e3:.1f} ms = {rows * F * 4 / dt / 1e9:.1f} GB/s uint32 read", flush=True)
    idv = cbk.id_vectors.cpu().numpy()
    val = cbk.value_vectors.cpu().numpy()
    etb = cbk.encode_tiebreak.cpu().numpy()
    mtb = cbk.model_tiebreak.cpu().numpy()
    outl = np.zeros(n_te, np.int32)
    ctx = eng.dc.ctx
    ctx.set_stream(None)
    p = lambda a: C.c_void_p(a.ctypes.data) if isinstance(a, np.ndarray) else C.c_void_p(a.data_ptr())
    for rep in range(4):
        f = C.c_void_p()
        t0 = time.perf_counter()
        N.check(L.hv_fold_encode_train(ctx.handle, p(b32), n_tr, p(lab), C.c_void_p(b32.data_ptr() + n_tr * F * 4),
                                       n_te, F, p(idv), p(val), B, D, p(etb), Cc, C.byref(f)))
        t1 = time.perf_counter()
        N.check(L.hv_fold_predict(ctx.handle, f, p(mtb), p(outl)))
        t2 = time.perf_counter()
        L.hv_fold_destroy(f)
        t3 = time.perf_counter()
        print(f"fold rep {rep}: encode_train {(t1 - t0) * 1e3:.2f} ms, predict {(t2 - t1) * 1e3:.2f} ms, "
              f"destroy {(t3 - t2) * 1e3:.2f} ms, total {(t3 - t0) * 1e3:.2f} ms = {rows / (t3 - t0) / 1e6:.2f} M dp/s",
              flush=True)
    eng.dc.bind()
    d8 = out8.cuda()
    enc = eng.pitched_empty(rows)
    for rep in range(3):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        eng.encode(d8, out=enc)
        b.record()
        torch.cuda.synchronize()
        print(f"resident encode of all rows: {a.elapsed_time(b):.2f} ms", flush=True)
    # the staging pipeline's device side without the host: the same chunking
    # (one stream / two alternating streams / two streams + pinned H2D per chunk)
    chunk = (32 << 20) // ldb
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    dbuf = [torch.empty((chunk, ldb), dtype=torch.uint8, device="cuda") for _ in range(2)]
    for mode in ("1 stream", "2 streams", "2 streams + H2D"):
        for rep in range(2):
            torch.cuda.synchronize()
            t = time.perf_counter()
            for k, r0 in enumerate(range(0, rows, chunk)):
                n = min(chunk, rows - r0)
                st = streams[k & 1] if mode != "1 stream" else streams[0]
                with torch.cuda.stream(st):
                    eng.dc.bind(st)
                    if mode.endswith("H2D"):
                        dbuf[k & 1][:n].copy_(out8[r0:r0 + n], non_blocking=True)
                        eng.encode(dbuf[k & 1][:n], out=enc[r0:r0 + n])
                    else:
                        eng.encode(d8[r0:r0 + n], out=enc[r0:r0 + n])
            torch.cuda.synchronize()
            print(f"chunked encode ({mode}, {chunk} rows per chunk): {(time.perf_counter() - t) * 1e3:.2f} ms",
                  flush=True)
    eng.dc.bind()


if __name__ == "__main__":
    main()
