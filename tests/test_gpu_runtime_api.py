"""The reference-shaped Python API (paper_2604_27058_b200.runtime) on the GPU.

Mirrors the reference's own hot-path tests (reference tests/test_runtime.py) on
programs restored from the golden fixtures: same records as the reference for
the same seed, post-selection semantics, error behaviour, live k.
"""
from __future__ import annotations

import math

import numpy as np
import pytest

from goldens import load
from paper_2604_27058_b200 import runtime as R

pytestmark = pytest.mark.gpu


def test_sample_reproduces_reference_records(cuda):
    for name in ("toy_noise_twice", "config1", "config2", "rand05"):
        g = load(name)
        recs = list(R.sample(g["prog"], g["f_meas"].shape[0], seed=int(g["f_seed"][0])))
        np.testing.assert_array_equal(np.array([r.measurements for r in recs]), g["f_meas"])


def test_mirror_deterministic(cuda):
    # reference test_runtime.py:36-41 (EXACT_MIRROR, 3000 shots, all-zero records)
    P = load("toy_mirror")["prog"]
    b = R.sample_batch(P, 3000, seed=0)
    assert not b["measurements"].any()
    b = R.Sampler(P, rng="philox").sample_batch(100_000, seed=1)
    assert not b["measurements"].any()


def test_h_t_h_branch_probability(cuda):
    # reference test_runtime.py:53-59
    P = load("toy_htm")["prog"]
    n = 2_000_000
    acc = R.Sampler(P, rng="philox").accumulate(n, seed=3)
    p = acc["measurements"][0] / n
    e = math.sin(math.pi / 8) ** 2
    assert abs(p - e) < 4 * math.sqrt(e * (1 - e) / n)


def test_postselect_rejection_and_filtering(cuda):
    # reference test_runtime.py:307-316 / :388-392
    P = load("toy_postselect1")["prog"]
    recs = list(R.sample(P, 2000, seed=12, keep_rejected=False))
    assert recs and all(r.measurements[0] == 1 for r in recs)
    assert abs(len(recs) / 2000 - 0.5) < 0.06
    allr = list(R.sample(P, 2000, seed=12, keep_rejected=True))
    assert len(allr) == 2000


def test_sample_requires_positive_shots(cuda):
    with pytest.raises(ValueError):
        list(R.sample(load("toy_htm")["prog"], 0))


def test_forced_zero_probability_branch_raises(cuda):
    # reference test_runtime.py:268-271: "M 0" forced to 1 is impossible
    P = load("toy_htm")["prog"]  # H T H M: outcome 1 has p = sin^2(pi/8) > 0; force via record on a static
    Q = load("toy_mirror")["prog"]  # deterministic all-zero records
    with pytest.raises(R.ShotError, match="probability"):
        R.run_shot(Q, shot=0, forced_outcomes={0: 1})
    R.run_shot(P, shot=0, forced_outcomes={0: 1})  # possible: no error


def test_run_shot_trace_k_tracks_schedule(cuda):
    # reference test_runtime.py:478-493
    for name in ("rand09", "bigk03"):
        P = load(name)["prog"]
        st = R.ShotState(P)
        seen = []
        R.run_shot(P, st, shot=3, trace=lambda s, _i: seen.append(s.k))
        assert seen == P.schedule.tolist()


def test_run_shot_forced_matches_reference(cuda):
    g = load("bigk02")
    P = g["prog"]
    for s in range(g["t_modes"].shape[0]):
        st = R.ShotState(P, seed=int(g["t_seed"][0]))
        fo = {r: int(v) for r, v in enumerate(g["t_forced"][s]) if v >= 0}
        rec = R.run_shot(P, st, shot=s, forced_faults=g["t_modes"][s], forced_outcomes=fo)
        np.testing.assert_array_equal(rec.measurements, g["t_meas"][s])
        np.testing.assert_array_equal(st.frame_x, g["t_fx"][s])
        assert abs(st.gamma - g["t_gamma"][s]) < 1e-10 * max(1.0, abs(g["t_gamma"][s]))


def test_gamma_squared_is_branch_probability(cuda):
    # reference test_runtime.py:252-256: "H 0; M 0; H 0; M 0" has two fair branches -> |gamma|^2 = 1/4
    from goldens import load_renorm

    P = load_renorm("two_fair")["prog"]
    for shot in range(8):
        st = R.ShotState(P)
        R.run_shot(P, st, shot=shot)
        assert abs(abs(st.gamma) ** 2 - 0.25) < 1e-12


def test_subnormalized_mode_tracks_branch_probability(cuda):
    # reference test_runtime.py:244-249: renormalize=False keeps |gamma|^2 ||phi||^2 = 1/4
    from goldens import load_renorm

    P = load_renorm("two_fair")["prog"]
    for shot in range(8):
        st = R.ShotState(P, renormalize=False)
        R.run_shot(P, st, shot=shot)
        total = abs(st.gamma) ** 2 * float(np.linalg.norm(st.active_view()) ** 2)
        assert abs(total - 0.25) < 1e-12


def test_sample_accumulate_matches_reference_marginals(cuda):
    g = load("config2")
    P = g["prog"]
    acc = R.sample_accumulate(P, g["f_meas"].shape[0], seed=int(g["f_seed"][0]))
    np.testing.assert_array_equal(acc["measurements"], g["f_meas"].sum(0))
    np.testing.assert_array_equal(acc["detectors"], g["f_det"].sum(0))
