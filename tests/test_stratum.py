"""Stratified importance sampling (runtime.py:886-945) against the reference.

Goldens (tests/golden/stratum/*.npz, tests/golden/make_golden.py "stratum") hold the reference's
``sample(prog, 96, seed=5, stratum=StratumSpec(prog, w))`` records and ``StratumSpec.weight`` for
w in {0, 1, 2, 3, 5}, the ValueError text for w > E, and ``framesim sample --format csv
--stratum-w`` bytes.  The reference stream (FS_RNG_SPLITMIX) must match bit for bit; the
engine stream is compared bit for bit with the oracle's restatement.
"""
from __future__ import annotations

import io
from pathlib import Path

import numpy as np
import pytest

import oracle
from paper_2604_27058_b200._abi import FS_RNG_PHILOX, FS_RNG_SPLITMIX
from paper_2604_27058_b200.program import Program

SDIR = Path(__file__).parent / "golden" / "stratum"
CASES = sorted(p.stem for p in SDIR.glob("*.npz"))


def _load(name):
    with np.load(SDIR / f"{name}.npz", allow_pickle=False) as z:
        g = {k: z[k] for k in z.files}
    g["prog"] = Program.load(io.BytesIO(g["program"].tobytes()))
    return g


def _pairs():
    return [(c, int(w)) for c in CASES for w in _load(c)["ws"]]


def _check(out, g, w):
    np.testing.assert_array_equal(out.measurements(), g[f"w{w}_meas"])
    np.testing.assert_array_equal(out.detectors(), g[f"w{w}_det"])
    np.testing.assert_array_equal(out.observables(), g[f"w{w}_obs"])
    np.testing.assert_array_equal(out.accepted_bits(), g[f"w{w}_acc"])


def test_stratum_goldens_present():
    assert len(CASES) >= 6


@pytest.mark.parametrize("name,w", _pairs())
def test_oracle_stratum_weight_matches_reference(name, w):
    g = _load(name)
    assert oracle.stratum_weight(g["prog"], w) == float(g[f"w{w}_weight"][0])


@pytest.mark.parametrize("name,w", _pairs())
def test_oracle_stratum_records_match_reference(name, w):
    g = _load(name)
    n = g[f"w{w}_acc"].shape[0]
    st, out = oracle.sample_stratum(g["prog"], w, n, seed=5, flags=FS_RNG_SPLITMIX)
    _check(out, g, w)


@pytest.mark.parametrize("name", [c for c in CASES if "too_many_error" in _load(c)])
def test_stratum_too_many_faults_error(name):
    from paper_2604_27058_b200.runtime import StratumSpec

    g = _load(name)
    with pytest.raises(ValueError) as ei:
        StratumSpec(g["prog"], g["prog"].num_sites + 1)
    assert str(ei.value) == str(g["too_many_error"])


@pytest.mark.parametrize("name", [c for c in CASES if "cli_csv" in _load(c)])
def test_oracle_stratum_csv_matches_reference_cli(name):
    g = _load(name)
    w = int(g["cli_w"][0])
    n = g[f"w{w}_acc"].shape[0]
    _, out = oracle.sample_stratum(g["prog"], w, n, seed=5, flags=FS_RNG_SPLITMIX)
    body = oracle.format_records(out.measurements(), out.detectors(), out.observables(),
                                 out.accepted_bits().astype(bool), "csv", True,
                                 weight=oracle.stratum_weight(g["prog"], w))
    assert b"shot,weight,bits\n" + body == g["cli_csv"].tobytes()


# ----------------------------------------------------------------------------- GPU
@pytest.mark.gpu
@pytest.mark.parametrize("name,w", _pairs())
@pytest.mark.parametrize("chunk", [None, "64"])
def test_gpu_stratum_matches_reference(cuda, name, w, chunk, monkeypatch):
    from paper_2604_27058_b200.engine import DeviceProgram

    if chunk:
        monkeypatch.setenv("FS_STRATUM_CHUNK", chunk)
    g = _load(name)
    dp = DeviceProgram(g["prog"])
    assert dp.stratum_weight(w) == float(g[f"w{w}_weight"][0])
    n = g[f"w{w}_acc"].shape[0]
    _, out = dp.sample_stratum_host(w, n, seed=5, flags=FS_RNG_SPLITMIX)
    _check(out, g, w)


@pytest.mark.gpu
@pytest.mark.parametrize("name,w", [p for p in _pairs() if p[1] > 0])
def test_gpu_stratum_philox_matches_oracle(cuda, name, w, monkeypatch):
    from paper_2604_27058_b200.engine import DeviceProgram

    monkeypatch.setenv("FS_STRATUM_CHUNK", "4096")
    g = _load(name)
    dp = DeviceProgram(g["prog"])
    n = 10_000
    _, a = dp.sample_stratum_host(w, n, seed=9, shot0=64, flags=FS_RNG_PHILOX)
    _, b = oracle.sample_stratum(g["prog"], w, n, seed=9, shot0=64, flags=FS_RNG_PHILOX)
    np.testing.assert_array_equal(a.measurements(), b.measurements())
    np.testing.assert_array_equal(a.detectors(), b.detectors())
    np.testing.assert_array_equal(a.observables(), b.observables())
    np.testing.assert_array_equal(a.accepted_bits(), b.accepted_bits())


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_gpu_runtime_importance_sample(cuda, name):
    from paper_2604_27058_b200 import runtime

    g = _load(name)
    w = int(g["ws"][-1])
    n = g[f"w{w}_acc"].shape[0]
    recs = list(runtime.importance_sample(g["prog"], w, n, seed=5))
    assert [r.accepted for r in recs] == [bool(x) for x in g[f"w{w}_acc"]]
    assert all(r.weight == float(g[f"w{w}_weight"][0]) for r in recs)
    np.testing.assert_array_equal(np.array([r.measurements for r in recs]).reshape(n, -1), g[f"w{w}_meas"])
    acc = runtime.sample_accumulate(g["prog"], n, seed=5, stratum=runtime.StratumSpec(g["prog"], w))
    a = g[f"w{w}_acc"].astype(bool)
    assert acc["accepted"] == int(a.sum())
    np.testing.assert_array_equal(acc["measurements"], g[f"w{w}_meas"][a].sum(0))
    np.testing.assert_array_equal(acc["detectors"], g[f"w{w}_det"][a].sum(0))
    wsum = 0.0
    for _ in range(int(a.sum())):
        wsum += float(g[f"w{w}_weight"][0])
    assert acc["weight_sum"] == wsum


@pytest.mark.gpu
@pytest.mark.parametrize("name", [c for c in CASES if "cli_csv" in _load(c)])
def test_gpu_stratum_csv_matches_reference_cli(cuda, name):
    from paper_2604_27058_b200 import runtime

    g = _load(name)
    w = int(g["cli_w"][0])
    n = g[f"w{w}_acc"].shape[0]
    got = runtime.sample_formatted(g["prog"], n, seed=5, format="csv", keep_rejected=True, stratum=w)
    assert got == g["cli_csv"].tobytes()
