"""Dataset-resident fold benchmark (hv_dataset_fold): upload fp64 features once, then time folds that fit the
discretizer, discretize, encode, train and predict on device. usage: python scripts/bench_dataset_fold.py"""
import sys, time, numpy as np, torch
sys.path.insert(0, '.')
from paper_2206_04746_b200 import hypervec as hv
n, F, C, B, D = 2_000_000, 342, 2, 16, 10000
rng = np.random.default_rng(0)
y = (rng.random(n) < 0.003).astype(np.int32)
X = rng.normal(size=(n, F)).astype(np.float64) + y[:, None] * 0.5
t0 = time.perf_counter(); ds = hv.Dataset(X, y); t1 = time.perf_counter()
print(f"dataset upload: {X.nbytes/1e9:.2f} GB in {t1-t0:.3f} s = {X.nbytes/(t1-t0)/1e9:.1f} GB/s")
cb = hv.make_codebook(0, 0, F, B, D, hv.derive_seed(1, 1)); etb = hv.generate_random(1, D, hv.derive_seed(1, 2))
cfg = hv.ModelConfig(class_count=C, dim=D, seed=1)
ntr = n * 4 // 5
tr, te = np.arange(ntr), np.arange(ntr, n)
for trainer in ("classical", "online"):
    ds.fold(tr, te, cb, etb, cfg, trainer, 1024)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(2):
        labels, mn, mx = ds.fold(tr, te, cb, etb, cfg, trainer, 1024)
    t = (time.perf_counter() - t0) / 2
    print(f"fold ({trainer}) from resident fp64 features: {t*1e3:.1f} ms = {n/t/1e6:.2f} M dp/s")
