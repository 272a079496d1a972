"""Degenerate programs and ragged shot counts, through every engine.

Goldens (tests/golden/edges, make_golden.py "edges"): programs the reference accepts with zero
instructions, zero records, noise with nothing measured, empty detectors / observables, an
unmeasured active array, 300 qubits with two touched; each with the reference's own
``sample(prog, 100, seed=9)`` records.
"""
from __future__ import annotations

import io
from pathlib import Path

import numpy as np
import pytest

import oracle
from goldens import load
from paper_2604_27058_b200._abi import (FS_FORCE_GENERAL, FS_FORCE_HBM, FS_NO_JIT, FS_RNG_PHILOX,
                                        FS_RNG_SPLITMIX)
from paper_2604_27058_b200.program import Program

EDIR = Path(__file__).parent / "golden" / "edges"
EDGES = sorted(p.stem for p in EDIR.glob("*.npz"))


def _edge(name):
    with np.load(EDIR / f"{name}.npz", allow_pickle=False) as z:
        g = {k: z[k] for k in z.files}
    g["prog"] = Program.load(io.BytesIO(g["program"].tobytes()))
    return g


def _same(a, b):
    np.testing.assert_array_equal(a.measurements(), b.measurements())
    np.testing.assert_array_equal(a.detectors(), b.detectors())
    np.testing.assert_array_equal(a.observables(), b.observables())
    np.testing.assert_array_equal(a.accepted_bits(), b.accepted_bits())


@pytest.mark.parametrize("name", EDGES)
def test_oracle_edges_match_reference(name):
    g = _edge(name)
    _, out, _ = oracle.sample(g["prog"], 100, seed=9, flags=FS_RNG_SPLITMIX)
    np.testing.assert_array_equal(out.measurements(), g["f_meas"])
    np.testing.assert_array_equal(out.detectors(), g["f_det"])
    np.testing.assert_array_equal(out.observables(), g["f_obs"])
    np.testing.assert_array_equal(out.accepted_bits(), g["f_acc"])


@pytest.mark.gpu
@pytest.mark.parametrize("name", EDGES)
@pytest.mark.parametrize("extra", [0, FS_FORCE_GENERAL, FS_FORCE_HBM])
def test_gpu_edges_match_reference(cuda, name, extra):
    from paper_2604_27058_b200.engine import DeviceProgram

    g = _edge(name)
    dp = DeviceProgram(g["prog"])
    _, out, _ = dp.sample_host(100, seed=9, flags=FS_RNG_SPLITMIX | extra)
    np.testing.assert_array_equal(out.measurements(), g["f_meas"])
    np.testing.assert_array_equal(out.detectors(), g["f_det"])
    np.testing.assert_array_equal(out.observables(), g["f_obs"])
    np.testing.assert_array_equal(out.accepted_bits(), g["f_acc"])


@pytest.mark.gpu
@pytest.mark.parametrize("name", EDGES)
@pytest.mark.parametrize("extra", [0, FS_NO_JIT, FS_FORCE_GENERAL, FS_FORCE_HBM])
def test_gpu_edges_philox_match_oracle(cuda, name, extra):
    from paper_2604_27058_b200.engine import DeviceProgram

    g = _edge(name)
    dp = DeviceProgram(g["prog"])
    _, a, _ = dp.sample_host(1000, seed=2**64 - 1, shot0=2**40, flags=FS_RNG_PHILOX | extra)
    _, b, _ = oracle.sample(g["prog"], 1000, seed=2**64 - 1, shot0=2**40, flags=FS_RNG_PHILOX)
    _same(a, b)


RAGGED = [1, 31, 33, 4097, 100_003]


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["config1", "config2", "config4", "toy_repetition", "bigk03"])
@pytest.mark.parametrize("n", RAGGED)
def test_gpu_ragged_shot_counts_match_oracle(cuda, name, n):
    """Shot counts that are not multiples of 32 (partial last word) on the default engine of each
    program: frame JIT (config1), general JIT (config2), segmented (config4), general, ..."""
    from paper_2604_27058_b200.engine import DeviceProgram

    P = load(name)["prog"]
    if n > 10_000 and name in ("config4", "bigk03"):
        n = 10_001
    dp = DeviceProgram(P)
    _, a, _ = dp.sample_host(n, seed=17, shot0=96, flags=FS_RNG_PHILOX)
    _, b, _ = oracle.sample(P, n, seed=17, shot0=96, flags=FS_RNG_PHILOX)
    _same(a, b)
    acc = dp.accumulate(n, seed=17, shot0=96, flags=FS_RNG_PHILOX)
    keep = b.accepted_bits().astype(bool)
    assert acc["accepted"] == int(keep.sum())
    np.testing.assert_array_equal(acc["measurements"], b.measurements()[keep].sum(0))
