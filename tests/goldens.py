"""Loader for the reference-generated fixtures in tests/golden (see make_golden.py)."""
from __future__ import annotations

import io
from functools import lru_cache
from pathlib import Path

import numpy as np

from paper_2604_27058_b200.program import Program

GOLDEN = Path(__file__).resolve().parent / "golden"


def case_names(prefix: str = "") -> list[str]:
    return sorted(p.stem for p in GOLDEN.glob(f"{prefix}*.npz"))


@lru_cache(maxsize=None)
def load(name: str) -> dict:
    with np.load(GOLDEN / f"{name}.npz", allow_pickle=False) as z:
        d = {k: z[k] for k in z.files}
    d["prog"] = Program.load(io.BytesIO(d["program"].tobytes()))
    return d


def rel_err(a, b) -> float:
    a = np.asarray(a)
    b = np.asarray(b)
    den = max(float(np.linalg.norm(b)), 1e-300)
    return float(np.linalg.norm(a - b)) / den
