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


def _load_path(path: Path) -> dict:
    with np.load(path, allow_pickle=False) as z:
        d = {k: z[k] for k in z.files}
    if "program" in d:
        d["prog"] = Program.load(io.BytesIO(d["program"].tobytes()))
    return d


@lru_cache(maxsize=None)
def load_renorm(name: str) -> dict:
    """renormalize=False fixtures (make_golden.py "renorm")."""
    return _load_path(GOLDEN / "renorm" / f"{name}.npz")


def renorm_names() -> list[str]:
    return sorted(p.stem for p in (GOLDEN / "renorm").glob("*.npz"))


@lru_cache(maxsize=None)
def load_deep(name: str) -> dict:
    """Deep trace fixtures with sketched checkpoints (make_golden.py "c3deep" / "c4deep")."""
    return _load_path(GOLDEN / "deep" / f"{name}.npz")


@lru_cache(maxsize=None)
def load_accept() -> list[dict]:
    """The 200 forced-trajectory circuits of the reference's acceptance criterion 3."""
    with np.load(GOLDEN / "accept" / "criterion3.npz", allow_pickle=False) as z:
        raw = {k: z[k] for k in z.files}
    out = []
    for i in range(200):
        key = f"c{i:03d}_"
        d = {k[len(key):]: v for k, v in raw.items() if k.startswith(key)}
        d["prog"] = Program.load(io.BytesIO(d["program"].tobytes()))
        out.append(d)
    return out


def sketch_vectors(k: int, seed: int, nvec: int, nent: int):
    """make_golden.sketch_vectors: fixed seeded complex vectors + sampled entry indices."""
    vecs = []
    for i in range(nvec):
        g = np.random.default_rng(seed + i)
        vecs.append(g.standard_normal(1 << k) + 1j * g.standard_normal(1 << k))
    idx = np.sort(np.random.default_rng(seed - 1).choice(1 << k, size=min(nent, 1 << k), replace=False))
    return vecs, idx


def frameref_names() -> list[str]:
    return sorted(p.stem for p in (GOLDEN / "frameref").glob("*.npz"))


@lru_cache(maxsize=None)
def load_frameref(name: str) -> dict:
    """Detector / observable counts of the reference's independent Pauli-frame sampler
    (framesim/oracle.py:407-516) for a Clifford program (make_golden.py "frameref")."""
    return _load_path(GOLDEN / "frameref" / f"{name}.npz")


@lru_cache(maxsize=None)
def load_mirrors50() -> list:
    """The 50 exact mirror programs of the reference's acceptance criterion 2."""
    with np.load(GOLDEN / "accept" / "criterion2_mirrors.npz", allow_pickle=False) as z:
        return [Program.load(io.BytesIO(z[k].tobytes())) for k in sorted(z.files)]


def max_two_sample_z(a, b, na: int, nb: int) -> float:
    """Largest two-sample binomial |z| (pooled sigma, each side's own n) over paired counts
    (test_acceptance.py:163-169)."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    p = (a + b) / (na + nb)
    sig = np.sqrt(np.maximum(p * (1 - p), 1e-12) * (1.0 / na + 1.0 / nb))
    return float(np.max(np.abs(a / na - b / nb) / sig)) if a.size else 0.0
