"""CPU: the oracle (test infrastructure) against the round-2 reference fixtures.

* ``accept.npz`` -- the 200 forced-trajectory circuits of the reference's acceptance criterion 3
  (pkg/tests/test_acceptance.py:131-152): every record (hidden ones included), detector,
  observable and frame bit-exact, gamma and the final active array within 1e-10; the reference's
  records there equal its dense oracle's (the criterion itself);
* ``renorm/*`` -- renormalize=False (runtime.py:355-366, :389-404, :481): free sampling with the
  reference stream bit-exact, and the unnormalised states of free shots (gamma,
  |gamma|^2 ||phi||^2, records, frames, amplitudes);
* ``deep/config4_deep`` -- accepted config-4 trajectories (all 15 post-selections pass): final
  state and the sketched checkpoints at k >= 10;
* ``frameref/*`` -- detector / observable rates against the reference's independent Pauli-frame
  sampler (oracle.py:407-516; config 1, a boosted surface code, criterion 4's repetition code).
"""
from __future__ import annotations

import numpy as np
import pytest

import oracle
from goldens import (frameref_names, load_accept, load_deep, load_frameref, load_renorm, max_two_sample_z,
                     rel_err, renorm_names, sketch_vectors)
from paper_2604_27058_b200._abi import FS_NO_RENORM, FS_RNG_SPLITMIX

TOL = 1e-10


def _modes(d):
    m = d["modes"]
    return None if m.size == 0 else m[None, :]


@pytest.mark.parametrize("chunk", range(4))
def test_oracle_matches_acceptance_trajectories(chunk):
    cases = load_accept()[chunk * 50:(chunk + 1) * 50]
    for i, d in enumerate(cases):
        P = d["prog"]
        np.testing.assert_array_equal(d["meas"], d["oracle_meas"][: d["meas"].size])  # criterion 3 itself
        st, out, tb = oracle.sample(P, 1, seed=int(d["seed"][0]), flags=FS_RNG_SPLITMIX, fault_modes=_modes(d),
                                    forced=d["forced"][None, :], want_state=True)
        assert st == 0, i
        np.testing.assert_array_equal(out.measurements()[0], d["meas"])
        np.testing.assert_array_equal(out.detectors()[0], d["det"])
        np.testing.assert_array_equal(out.observables()[0], d["obs"])
        np.testing.assert_array_equal(tb.records[0, :P.record_count], d["rec"])
        np.testing.assert_array_equal(tb.frame_x[0, :P.n], d["fx"])
        np.testing.assert_array_equal(tb.frame_z[0, :P.n], d["fz"])
        assert rel_err(tb.gamma_c()[:1], d["gamma"]) < TOL
        assert rel_err(tb.amps_c()[0], d["amps"]) < TOL


@pytest.mark.parametrize("name", renorm_names())
def test_oracle_renormalize_false(name):
    g = load_renorm(name)
    P = g["prog"]
    n = g["f_meas"].shape[0]
    st, out, _ = oracle.sample(P, n, seed=int(g["f_seed"][0]), flags=FS_RNG_SPLITMIX | FS_NO_RENORM)
    assert st == 0
    np.testing.assert_array_equal(out.measurements(), g["f_meas"])
    np.testing.assert_array_equal(out.detectors(), g["f_det"])
    np.testing.assert_array_equal(out.accepted_bits(), g["f_acc"])
    ns = g["s_gamma"].shape[0]
    st, out, tb = oracle.sample(P, ns, seed=int(g["s_seed"][0]), flags=FS_RNG_SPLITMIX | FS_NO_RENORM,
                                want_state=True)
    assert st == 0
    assert rel_err(tb.gamma_c(), g["s_gamma"]) < TOL
    total = np.abs(tb.gamma_c()) ** 2 * np.linalg.norm(tb.amps_c(), axis=1) ** 2
    np.testing.assert_allclose(total, g["s_total"], rtol=TOL, atol=0)
    np.testing.assert_array_equal(tb.records[:, :P.record_count], g["s_rec"])
    np.testing.assert_array_equal(tb.frame_x[:, :P.n], g["s_fx"])
    if "s_amps" in g:
        assert rel_err(tb.amps_c(), g["s_amps"]) < TOL
    if name == "two_fair":  # reference test_runtime.py:244-249
        np.testing.assert_allclose(total, 0.25, atol=1e-12)


def check_sketch(amps, g, c, valid):
    """amps [shots][2^k] against the fixture's sketch of checkpoint c (rows where valid)."""
    seed, nvec, nent = (int(x) for x in g["sk_seed"])
    k = int(np.log2(amps.shape[1]))
    vecs, idx = sketch_vectors(k, seed, nvec, nent)
    np.testing.assert_array_equal(idx, g[f"sk{c}_idx"])
    a = amps[valid]
    n2 = np.einsum("ij,ij->i", a.conj(), a).real
    np.testing.assert_allclose(n2, g[f"sk{c}_norm2"][valid], rtol=TOL, atol=0)
    ip = np.stack([a @ v.conj() for v in vecs], axis=1)
    assert rel_err(ip, g[f"sk{c}_ip"][valid]) < TOL
    assert rel_err(a[:, idx], g[f"sk{c}_vals"][valid]) < TOL


def test_oracle_config4_deep_trajectories():
    g = load_deep("config4_deep")
    P = g["prog"]
    n = g["t_modes"].shape[0]
    assert g["t_acc"].all()
    st, out, tb = oracle.sample(P, n, seed=int(g["t_seed"][0]), flags=FS_RNG_SPLITMIX, fault_modes=g["t_modes"],
                                forced=g["t_forced"], want_state=True)
    assert st == 0
    np.testing.assert_array_equal(out.measurements(), g["t_meas"])
    np.testing.assert_array_equal(out.detectors(), g["t_det"])
    np.testing.assert_array_equal(out.accepted_bits(), g["t_acc"])
    np.testing.assert_array_equal(tb.records[:, :P.record_count], g["t_rec"])
    np.testing.assert_array_equal(tb.frame_x[:, :P.n], g["t_fx"])
    assert rel_err(tb.gamma_c(), g["t_gamma"]) < TOL
    assert rel_err(tb.amps_c(), g["t_amps"]) < TOL
    for c in g["sk_index"].tolist():
        st, out, tb = oracle.sample(P, n, seed=int(g["t_seed"][0]), flags=FS_RNG_SPLITMIX, fault_modes=g["t_modes"],
                                    forced=g["t_forced"], stop=c + 1, want_state=True)
        valid = ~np.isnan(g[f"sk{c}_gamma"])
        assert valid.all()
        np.testing.assert_array_equal(tb.frame_x[:, :P.n], g[f"sk{c}_fx"])
        assert rel_err(tb.gamma_c(), g[f"sk{c}_gamma"]) < TOL
        check_sketch(tb.amps_c(), g, c, valid)


@pytest.mark.parametrize("name", frameref_names())
def test_oracle_rates_match_reference_frame_sampler(name):
    """The reference VM (oracle restatement, reference stream) vs the reference's independent
    Pauli-frame sampler (oracle.py:407-516): every detector / observable rate within 5 sigma
    (the config-1 check; acceptance criterion 4 for the repetition code)."""
    g = load_frameref(name)
    P = g["prog"]
    n = 200_000
    st, acc = oracle.accumulate(P, n, seed=77, flags=FS_RNG_SPLITMIX)
    assert st == 0
    ns = int(g["shots"][0])
    assert max_two_sample_z(acc["detectors"], g["det_counts"], n, ns) < 5.0
    assert max_two_sample_z(acc["observables"], g["obs_counts"], n, ns) < 5.0
