"""Workload for the source-level ncu capture of the online trainer at the
CHB-MIT shape (profiles/ncu_online_E_r2_late.txt):

  ncu --set full --import-source on --clock-control none -k regex:online_persistent_kernel -c 1 \\
      -o onl_e python scripts/online_ncu_E.py
"""
import os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_2206_04746_b200 import device as dv
cbk = dv.DeviceCodebook.make(342, 16, 10000, seed=3)
eng = dv.Engine(cbk, 2)
b8, y = eng.synth(0, 60_000, 1, 7)
enc = eng.encode(b8)
torch.cuda.synchronize()
eng.train_online(enc, y, 1024); torch.cuda.synchronize()
