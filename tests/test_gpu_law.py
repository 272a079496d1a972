"""Free-sampling LAW of the engine stream (FS_RNG_PHILOX) -- north_star: "5 sigma in free mode".

The Philox stream is checked bit for bit against the oracle elsewhere; that pins the
implementation, not the law.  Here:
  * every marginal (user records, detectors, observables) and the acceptance rate of the engine
    stream against the reference stream (FS_RNG_SPLITMIX, itself bit-identical to
    framesim.sample), two-sample binomial z with pooled sigma, |z| < 5 (SURVEY §8(d),
    test_acceptance.py:163-169);
  * the reference tests' known-answer laws (tests/golden/laws, compiled by the reference).
"""
from __future__ import annotations

import io
import math
from pathlib import Path

import numpy as np
import pytest

from goldens import load
from paper_2604_27058_b200._abi import FS_RNG_PHILOX, FS_RNG_SPLITMIX
from paper_2604_27058_b200.program import Program

pytestmark = pytest.mark.gpu
LDIR = Path(__file__).parent / "golden" / "laws"
PROGS = Path(__file__).resolve().parent.parent / "paper_2604_27058_b200" / "programs"
Z_MAX = 5.0


def _z(k1, n1, k2, n2):
    p = (k1 + k2) / (n1 + n2)
    se = math.sqrt(max(p * (1 - p) * (1 / n1 + 1 / n2), 0.0))
    if se == 0.0:
        return 0.0 if k1 / n1 == k2 / n2 else math.inf
    return (k1 / n1 - k2 / n2) / se


def _z1(k, n, p):
    se = math.sqrt(p * (1 - p) / n)
    if se == 0.0:
        return 0.0 if k / n == p else math.inf
    return (k / n - p) / se


def _acc(dp, n, flags):
    return dp.accumulate(n, seed=12345, flags=flags)


def _two_sample(P, n):
    from paper_2604_27058_b200.engine import DeviceProgram

    dp = DeviceProgram(P)
    a = _acc(dp, n, FS_RNG_PHILOX)
    b = _acc(dp, n, FS_RNG_SPLITMIX)
    worst = 0.0
    assert abs(_z(a["accepted"], n, b["accepted"], n)) < Z_MAX
    na, nb = max(a["accepted"], 1), max(b["accepted"], 1)
    for key in ("measurements", "detectors", "observables"):
        for ka, kb in zip(a[key], b[key]):
            z = _z(int(ka), na, int(kb), nb)
            worst = max(worst, abs(z))
            assert abs(z) < Z_MAX, (key, int(ka), na, int(kb), nb, z)
    return worst


@pytest.mark.parametrize("cfg,n", [(0, 400_000), (1, 1_000_000), (2, 1_000_000), (4, 4_000_000)])
def test_engine_stream_law_matches_reference_stream_configs(cuda, cfg, n):
    _two_sample(Program.load(PROGS / f"c{cfg}.npz"), n)


@pytest.mark.parametrize("name", ["toy_repetition", "toy_worked", "toy_feedforward", "toy_noise_twice",
                                  "toy_postselect", "rand03", "rand07", "rand11", "bigk02", "bigk06"])
def test_engine_stream_law_matches_reference_stream_goldens(cuda, name):
    _two_sample(load(name)["prog"], 300_000)


def _law(name):
    with np.load(LDIR / f"{name}.npz", allow_pickle=False) as z:
        return Program.load(io.BytesIO(z["program"].tobytes()))


def _samples(name, n, flags=FS_RNG_PHILOX):
    from paper_2604_27058_b200.engine import DeviceProgram

    dp = DeviceProgram(_law(name))
    _, out, _ = dp.sample_host(n, seed=777, flags=flags)
    return out


@pytest.mark.parametrize("flags", [FS_RNG_PHILOX, FS_RNG_SPLITMIX])
def test_law_htm_sin2_pi_8(cuda, flags):
    n = 400_000
    m = _samples("htm", n, flags).measurements()[:, 0]
    assert abs(_z1(int(m.sum()), n, math.sin(math.pi / 8) ** 2)) < Z_MAX


def test_law_fair_coin(cuda):
    n = 400_000
    m = _samples("coin", n).measurements()[:, 0]
    assert abs(_z1(int(m.sum()), n, 0.5)) < Z_MAX


def test_law_certain_sites(cuda):
    m = _samples("certain", 100_000).measurements()
    assert m[:, 0].all() and not m[:, 1].any()


def test_law_hazard_pair_joint(cuda):
    """Independent sites p = 0.1, 0.3: chi^2 of the four joint outcomes (3 dof) below its
    1e-6 quantile bound."""
    n = 400_000
    m = _samples("hazard_pair", n).measurements()
    cells = np.bincount(m[:, 0] * 2 + m[:, 1], minlength=4)
    p = np.array([0.9 * 0.7, 0.9 * 0.3, 0.1 * 0.7, 0.1 * 0.3])
    chi2 = float((((cells - n * p) ** 2) / (n * p)).sum())
    assert chi2 < 32.0  # chi^2_3 upper 1e-6 tail ~ 30.7


def test_law_fault_count_poisson_binomial(cuda):
    """test_acceptance.py:300-310: number of fired sites ~ Poisson-binomial(0.05, 0.2, 0.35, 0.5)."""
    n = 400_000
    m = _samples("pbinom", n).measurements()
    cnt = np.bincount(m.sum(1), minlength=5)
    pmf = np.array([1.0])
    for q in (0.05, 0.2, 0.35, 0.5):
        pmf = np.convolve(pmf, [1 - q, q])
    chi2 = float((((cnt - n * pmf) ** 2) / (n * pmf)).sum())
    assert chi2 < 36.0  # chi^2_4 upper 1e-6 tail ~ 33.4
    for q, col in zip((0.05, 0.2, 0.35, 0.5), m.T):
        assert abs(_z1(int(col.sum()), n, q)) < Z_MAX


def test_law_depolarize1(cuda):
    n = 400_000
    m = _samples("depol1", n).measurements()[:, 0]
    assert abs(_z1(int(m.sum()), n, 0.3 * 2 / 3)) < Z_MAX


def test_law_depolarize2_joint(cuda):
    """15 equiprobable Pauli pairs: (flip0, flip1) masses (1-p) + 3p/15, 4p/15, 4p/15, 4p/15."""
    n = 400_000
    pe = 0.15
    m = _samples("depol2", n).measurements()
    cells = np.bincount(m[:, 0] * 2 + m[:, 1], minlength=4)
    p = np.array([1 - pe + 3 * pe / 15, 4 * pe / 15, 4 * pe / 15, 4 * pe / 15])
    chi2 = float((((cells - n * p) ** 2) / (n * p)).sum())
    assert chi2 < 32.0


def test_law_postselect_acceptance_half(cuda):
    n = 400_000
    out = _samples("postselect_half", n)
    acc = out.accepted_bits().astype(bool)
    assert abs(_z1(int(acc.sum()), n, 0.5)) < Z_MAX
    m = out.measurements()[acc, 1]
    assert abs(_z1(int(m.sum()), int(acc.sum()), math.sin(math.pi / 8) ** 2)) < Z_MAX


def test_law_stratum_exact_fault_count(cuda):
    """Stratified sampling: exactly w of the four sites fire, in both streams, and the fired
    subsets follow the conditional law  P(S) ~ prod_{i in S} p_i prod_{i not in S} (1 - p_i)."""
    from itertools import combinations

    from paper_2604_27058_b200.engine import DeviceProgram

    qs = (0.05, 0.2, 0.35, 0.5)
    dp = DeviceProgram(_law("pbinom"))
    n = 300_000
    for flags in (FS_RNG_PHILOX, FS_RNG_SPLITMIX):
        for w in (1, 2, 3):
            _, out = dp.sample_stratum_host(w, n, seed=3, flags=flags)
            m = out.measurements()
            assert (m.sum(1) == w).all()
            subsets = list(combinations(range(4), w))
            weights = np.array([np.prod([qs[i] if i in S else 1 - qs[i] for i in range(4)]) for S in subsets])
            p = weights / weights.sum()
            code = (m * (1 << np.arange(4))).sum(1)
            idx = {sum(1 << i for i in S): k for k, S in enumerate(subsets)}
            cells = np.bincount([idx[c] for c in code], minlength=len(subsets))
            chi2 = float((((cells - n * p) ** 2) / (n * p)).sum())
            assert chi2 < 40.0, (flags, w, chi2)
