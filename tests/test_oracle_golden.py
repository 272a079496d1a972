"""Pin the CPU oracle (oracle/fs_oracle.c) to the REFERENCE implementation.

The fixtures in tests/golden were produced by the reference VM itself
(framesim.runtime, see tests/golden/make_golden.py).  The oracle must
reproduce them: records / detectors / observables / accepted bit-exact, in
trace mode and in free sampling with the reference SplitMix64 stream; frames
bit-exact; gamma and active amplitudes within 1e-10 relative (north_star).
"""
from __future__ import annotations

import numpy as np
import pytest

import oracle
from goldens import case_names, load, rel_err
from paper_2604_27058_b200._abi import FS_RNG_SPLITMIX

CASES = case_names()
AMP_TOL = 1e-10


def test_golden_fixtures_present():
    assert len(CASES) >= 40, CASES
    for prefix in ("toy_", "rand", "bigk", "mirror", "config"):
        assert any(c.startswith(prefix) for c in CASES), prefix


@pytest.mark.parametrize("name", [c for c in CASES if "f_meas" in load(c)])
def test_oracle_free_sampling_matches_reference(name):
    g = load(name)
    P = g["prog"]
    n = g["f_meas"].shape[0]
    st, out, _ = oracle.sample(P, n, seed=int(g["f_seed"][0]), flags=FS_RNG_SPLITMIX)
    assert st == 0
    np.testing.assert_array_equal(out.measurements(), g["f_meas"])
    np.testing.assert_array_equal(out.detectors(), g["f_det"])
    np.testing.assert_array_equal(out.observables(), g["f_obs"])
    np.testing.assert_array_equal(out.accepted_bits(), g["f_acc"])


@pytest.mark.parametrize("name", [c for c in CASES if "t_modes" in load(c)])
def test_oracle_trace_matches_reference(name):
    g = load(name)
    P = g["prog"]
    n = g["t_modes"].shape[0]
    st, out, tb = oracle.sample(P, n, seed=int(g["t_seed"][0]), flags=FS_RNG_SPLITMIX,
                                fault_modes=g["t_modes"], forced=g["t_forced"], want_state=True)
    assert st == 0
    np.testing.assert_array_equal(out.measurements(), g["t_meas"])
    np.testing.assert_array_equal(out.detectors(), g["t_det"])
    np.testing.assert_array_equal(out.observables(), g["t_obs"])
    np.testing.assert_array_equal(out.accepted_bits(), g["t_acc"])
    np.testing.assert_array_equal(tb.frame_x[:, :P.n], g["t_fx"])
    np.testing.assert_array_equal(tb.frame_z[:, :P.n], g["t_fz"])
    np.testing.assert_array_equal(tb.draws, g["t_draws"])
    assert rel_err(tb.gamma_c(), g["t_gamma"]) < AMP_TOL
    if "t_amps" in g and g["t_acc"].all():
        assert rel_err(tb.amps_c(), g["t_amps"]) < AMP_TOL


@pytest.mark.parametrize("name", [c for c in CASES if "cp_index" in load(c)])
def test_oracle_checkpoints_match_reference(name):
    g = load(name)
    P = g["prog"]
    n = g["t_modes"].shape[0]
    for c in g["cp_index"].tolist():
        st, out, tb = oracle.sample(P, n, seed=int(g["t_seed"][0]), flags=FS_RNG_SPLITMIX,
                                    fault_modes=g["t_modes"], forced=g["t_forced"], stop=c + 1,
                                    want_state=True)
        ok = ~np.isnan(g[f"cp{c}_gamma"])  # shots that halted before the checkpoint
        np.testing.assert_array_equal(tb.frame_x[ok, :P.n], g[f"cp{c}_fx"][ok])
        np.testing.assert_array_equal(tb.frame_z[ok, :P.n], g[f"cp{c}_fz"][ok])
        assert rel_err(tb.gamma_c()[ok], g[f"cp{c}_gamma"][ok]) < AMP_TOL
        assert rel_err(tb.amps_c()[ok], g[f"cp{c}_amps"][ok]) < AMP_TOL


def test_oracle_accumulate_is_sum_of_samples():
    g = load("toy_postselect")
    P = g["prog"]
    st, acc = oracle.accumulate(P, 5000, seed=4, flags=FS_RNG_SPLITMIX)
    st2, out, _ = oracle.sample(P, 5000, seed=4, flags=FS_RNG_SPLITMIX)
    a = out.accepted_bits().astype(bool)
    assert acc["accepted"] == a.sum()
    np.testing.assert_array_equal(acc["measurements"], out.measurements()[a].sum(0))
