"""Device output formats (fs_format) against the reference CLI's own bytes (cli.py:94-109).

Goldens: tests/golden/formats/*.npz, written by tests/golden/make_golden.py ("formats") by
running the reference ``framesim sample --format {01,bin,csv} [--keep-rejected]`` in-process.
"""
from __future__ import annotations

import io
from pathlib import Path

import numpy as np
import pytest

import oracle
from paper_2604_27058_b200._abi import FS_RNG_SPLITMIX
from paper_2604_27058_b200.program import Program

FDIR = Path(__file__).parent / "golden" / "formats"
CASES = sorted(p.stem for p in FDIR.glob("*.npz"))
FORMATS = ("01", "bin", "csv")


def _load(name):
    with np.load(FDIR / f"{name}.npz", allow_pickle=False) as z:
        g = {k: z[k] for k in z.files}
    g["prog"] = Program.load(io.BytesIO(g["program"].tobytes()))
    return g


def test_format_goldens_present():
    assert len(CASES) >= 5


@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("fmt", FORMATS)
@pytest.mark.parametrize("keep", [False, True])
def test_oracle_formatter_matches_reference_cli(name, fmt, keep):
    """The CPU checker reproduces the reference CLI bytes from the oracle's reference-stream run."""
    g = _load(name)
    n, seed = int(g["shots"][0]), int(g["seed"][0])
    _, out, _ = oracle.sample(g["prog"], n, seed=seed, flags=FS_RNG_SPLITMIX)
    body = oracle.format_records(out.measurements(), out.detectors(), out.observables(),
                                 out.accepted_bits().astype(bool), fmt, keep)
    if fmt == "csv":
        body = b"shot,weight,bits\n" + body
    assert body == g[f"{fmt}_{int(keep)}"].tobytes()


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("fmt", FORMATS)
@pytest.mark.parametrize("keep", [False, True])
@pytest.mark.parametrize("chunk", [1 << 20, 64])
def test_gpu_formatted_matches_reference_cli(cuda, name, fmt, keep, chunk):
    from paper_2604_27058_b200 import runtime

    g = _load(name)
    n, seed = int(g["shots"][0]), int(g["seed"][0])
    got = runtime.sample_formatted(g["prog"], n, seed=seed, format=fmt, keep_rejected=keep,
                                   rng="reference", chunk=chunk)
    assert got == g[f"{fmt}_{int(keep)}"].tobytes()


@pytest.mark.gpu
@pytest.mark.parametrize("fmt", FORMATS)
def test_gpu_formatted_philox_matches_oracle_large(cuda, fmt):
    """Engine stream, 200k shots in 4 chunks: device formatter == CPU restatement over the oracle."""
    from paper_2604_27058_b200 import runtime

    g = _load("surface_d3")
    n = 200_000
    got = runtime.sample_formatted(g["prog"], n, seed=3, format=fmt, keep_rejected=True, rng="philox",
                                   chunk=1 << 16)
    _, out, _ = oracle.sample(g["prog"], n, seed=3, flags=0)
    body = oracle.format_records(out.measurements(), out.detectors(), out.observables(),
                                 out.accepted_bits().astype(bool), fmt, True)
    if fmt == "csv":
        body = b"shot,weight,bits\n" + body
    assert got == body
