"""Worker bodies for the multi-process GPU tests (tests/test_gpu_multiproc.py).

Each worker is one rank of a `gloo` process group on 127.0.0.1; all ranks
share the visible GPU (the gpurun boxes have one). They run the engine's own
multi-GPU training paths — not NumPy restatements — and save their results
for the parent test to compare with the oracle.
"""
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def online_ranks(rank, world, port, out_dir, F, C, D, rows, bsz, seed, data_seed):
    import torch
    import torch.distributed as dist

    from paper_2206_04746_b200 import device as dv

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    cbk = dv.DeviceCodebook.make(F, 16, D, seed=seed)
    eng = dv.Engine(cbk, C)
    bins8, labels = eng.synth(0, rows, 0, data_seed)
    W = eng.W
    # exact word-sliced mode: the popcount all-reduce through torch.distributed (gloo)
    w0, nw = dv.word_slice(W, rank, world)
    sl = eng.encode_words(bins8, w0, nw)
    acc, weight, counts, cv = dv.DSlicedOnline(eng, sl, labels, bsz, w0).run()
    np.savez(os.path.join(out_dir, f"sliced_{rank}.npz"), acc=acc.cpu().numpy(), weight=weight.cpu().numpy(),
             counts=counts.cpu().numpy(), cv=cv.cpu().numpy(), w0=w0, nw=nw)
    # exact word-sliced mode with the all-reduce fused into the partial kernel over peer memory
    peers = dv.PeerPopc(eng, rank, world, bsz)
    for _ in range(2):  # reusing the peer buffers for a second run (epochs keep growing)
        acc2, _, _, cv2 = dv.DSlicedOnline(eng, sl, labels, bsz, w0).run(peers=peers)
    peers.close()
    np.savez(os.path.join(out_dir, f"peer_{rank}.npz"), acc=acc2.cpu().numpy(), cv=cv2.cpu().numpy())
    # delta mode: each rank owns a contiguous slice of every global batch
    idx = torch.as_tensor(dv.shard_rows_online(rows, bsz, rank, world), device=eng.dev)
    enc = eng.encode(bins8)
    acc3, w3, c3, cv3 = eng.train_online_sharded(enc[idx].contiguous(), labels[idx].contiguous(), rows, bsz, rank,
                                                 world)
    np.savez(os.path.join(out_dir, f"delta_{rank}.npz"), acc=acc3.cpu().numpy(), weight=w3.cpu().numpy(),
             counts=c3.cpu().numpy(), cv=cv3.cpu().numpy())
    if rank == 0:
        np.savez(os.path.join(out_dir, "inputs.npz"), enc=enc.cpu().numpy(), labels=labels.cpu().numpy(),
                 tiebreak=cbk.model_tiebreak.cpu().numpy())
    dist.barrier()
    dist.destroy_process_group()
