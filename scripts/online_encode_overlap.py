"""Timing only: the encoder and the online trainer launched concurrently on two
streams (the trainer on pre-encoded rows) at the CHB-MIT train-row shape, to
measure whether they co-schedule. usage: python scripts/online_encode_overlap.py
"""
import os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_2206_04746_b200 import device as dv
F, D, rows = 342, 10000, 5_648_000
cbk = dv.DeviceCodebook.make(F, 16, D, seed=3)
eng = dv.Engine(cbk, 2)
b8, y = eng.synth(0, rows, 1, 7)
W = eng.W
encA = torch.empty((rows, W), dtype=torch.int32, device='cuda')
encB = eng.encode_words(b8, 0, W)  # valid rows for the trainer
sB = torch.cuda.Stream()
eng2 = dv.Engine(cbk, 2)
def ev():
    return torch.cuda.Event(enable_timing=True)
def enc_only(shape):
    if shape: os.environ["HVB200_TT_SHAPE"] = shape
    else: os.environ.pop("HVB200_TT_SHAPE", None)
    eng.encode_words(b8, 0, W, out=encA); torch.cuda.synchronize()
    a, b = ev(), ev(); a.record(); eng.encode_words(b8, 0, W, out=encA); b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b)
def train_only():
    eng.train_online(encB, y, 1024); torch.cuda.synchronize()
    a, b = ev(), ev(); a.record(); eng.train_online(encB, y, 1024); b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b)
print("encode {3,12} alone", enc_only(None), flush=True)
for sh in ("2,8,1", "3,8,1", "2,12,1"):
    try:
        print("encode", sh, "alone", enc_only(sh), flush=True)
    except Exception as e:
        print(sh, e)
print("train alone", train_only(), flush=True)
for sh in ("2,8,1", "3,8,1"):
    os.environ["HVB200_TT_SHAPE"] = sh
    torch.cuda.synchronize()
    a = ev(); a.record()
    with torch.cuda.stream(sB):
        eng2.dc.bind(sB)
        sB.wait_event(a)
        eng2.train_online(encB, y, 1024)
        bB = ev(); bB.record(sB)
    eng.dc.bind()
    eng.encode_words(b8, 0, W, out=encA)
    bA = ev(); bA.record()
    torch.cuda.synchronize()
    print("concurrent", sh, "encode end", a.elapsed_time(bA), "train end", a.elapsed_time(bB), flush=True)
