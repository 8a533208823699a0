"""Loader for tests/golden/cases (written by oracle/golden_gen.cpp from the reference)."""
from __future__ import annotations

from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden" / "cases"


class Case:
    def __init__(self, name: str):
        self.name = name
        self.dir = GOLDEN / name
        if not self.dir.is_dir():
            raise FileNotFoundError(f"golden case {name} missing; run `make -C oracle golden`")
        self.meta = {}
        meta = self.dir / "meta.txt"
        if meta.exists():
            for line in meta.read_text().splitlines():
                k, _, v = line.partition("=")
                self.meta[k] = v

    def __getitem__(self, key: str) -> np.ndarray:
        return np.load(self.dir / f"{key}.npy")

    def has(self, key: str) -> bool:
        return (self.dir / f"{key}.npy").exists()

    def int(self, key: str) -> int:
        return int(self.meta[key])

    def float_bits(self, key: str) -> float:
        return float(np.array([int(self.meta[key])], dtype=np.uint64).view(np.float64)[0])


def cases(prefix: str):
    return sorted(p.name for p in GOLDEN.iterdir() if p.name.startswith(prefix))
