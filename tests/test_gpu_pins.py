"""GPU parity on the paths the benchmark times, against the round-2 reference fixtures.

* config 3 (k = 22, the large-k engine with the NVRTC fused passes the bench times): 8 trace
  shots, checkpoints at k >= 20 in ONE call (fs_trace_in.checkpoints), amplitude sketches within
  1e-10 of the reference, records / frames bit-exact; 5-sigma law of the Philox stream against
  the reference stream on all 22 marginals;
* config 4: accepted trajectories (all 15 post-selections pass) through the SEGMENTED engine
  (lane / warp / CTA-per-shot block kernels) and the general interpreter, checkpoints at
  k = 10-12 against reference amplitudes; Philox free sampling vs the oracle on 131,072 shots;
* the 200 forced trajectories of the reference's acceptance criterion 3, every engine;
* renormalize=False (free sampling + unnormalised states), every engine;
* ShotState.records holds hidden records too (trace outputs), vs reference and oracle;
* NaN injected into an Expand phase raises ShotError("NaN") on every engine (reference
  test_runtime.py:274-281), also through sample_accumulate;
* detector / observable rates vs the reference's independent Pauli-frame sampler (config 1, SURVEY
  §8(d); acceptance criterion 4) and the 50 exact mirrors of acceptance criterion 2.
"""
from __future__ import annotations

import math

import numpy as np
import pytest

import oracle
from goldens import (case_names, frameref_names, load, load_accept, load_deep, load_frameref, load_mirrors50,
                     load_renorm, max_two_sample_z, rel_err, renorm_names)
from paper_2604_27058_b200._abi import (FS_FORCE_GENERAL, FS_FORCE_HBM, FS_FORCE_SEGMENTED, FS_NO_JIT,
                                        FS_NO_RENORM, FS_RNG_PHILOX, FS_RNG_SPLITMIX)
from test_oracle_pins import check_sketch

pytestmark = pytest.mark.gpu
TOL = 1e-10


def _dev(P):
    from paper_2604_27058_b200.engine import DeviceProgram

    return DeviceProgram(P)


def _trace_all(dp, g, flags, checkpoints=None):
    n = g["t_modes"].shape[0]
    st, out, tb = dp.sample_host(n, seed=int(g["t_seed"][0]), flags=flags, fault_modes=g["t_modes"],
                                 forced=g["t_forced"], want_state=True, checkpoints=checkpoints)
    assert st == 0
    return out, tb


def _check_final(P, g, out, tb):
    np.testing.assert_array_equal(out.measurements(), g["t_meas"])
    np.testing.assert_array_equal(out.detectors(), g["t_det"])
    np.testing.assert_array_equal(out.observables(), g["t_obs"])
    np.testing.assert_array_equal(out.accepted_bits(), g["t_acc"])
    np.testing.assert_array_equal(tb.records[:, :P.record_count], g["t_rec"])
    np.testing.assert_array_equal(tb.frame_x[:, :P.n], g["t_fx"])
    np.testing.assert_array_equal(tb.frame_z[:, :P.n], g["t_fz"])
    assert rel_err(tb.gamma_c(), g["t_gamma"]) < TOL
    if "t_amps" in g:
        assert rel_err(tb.amps_c(), g["t_amps"]) < TOL


# ---------------------------------------------------------------------------- config 3
@pytest.mark.parametrize("env", [{}, {"FS_HBM_NO_JIT": "1"}, {"FS_PASS_TMA": "1"}])
def test_gpu_config3_trace_checkpoints_match_reference(cuda, env, monkeypatch):
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    g = load_deep("config3_deep")
    P = g["prog"]
    dp = _dev(P)
    assert dp.engine(0) == "hbm"
    cps = g["sk_index"].tolist()
    out, tb = _trace_all(dp, g, FS_RNG_PHILOX, checkpoints=[c + 1 for c in cps])
    _check_final(P, g, out, tb)
    for j, c in enumerate(cps):
        cp = tb.checkpoint(j)
        assert cp["valid"].all() and cp["k"] >= 20
        np.testing.assert_array_equal(cp["frame_x"], g[f"sk{c}_fx"])
        np.testing.assert_array_equal(cp["frame_z"], g[f"sk{c}_fz"])
        assert rel_err(cp["gamma"], g[f"sk{c}_gamma"]) < TOL
        check_sketch(cp["amps"], g, c, cp["valid"])


def _two_sample_z(a, b, na, nb):
    pa, pb = a / na, b / nb
    p = (a + b) / (na + nb)
    sig = math.sqrt(max(p * (1 - p), 1e-12) * (1 / na + 1 / nb))
    return abs(pa - pb) / sig


def test_gpu_config3_philox_law_vs_reference_stream(cuda):
    """5 sigma: every one of the 22 measurement marginals, Philox vs the reference stream."""
    P = load("config3")["prog"]
    dp = _dev(P)
    n = 2048
    a = dp.accumulate(n, seed=21, flags=FS_RNG_PHILOX)
    b = dp.accumulate(n, seed=22, flags=FS_RNG_SPLITMIX)
    assert a["accepted"] == b["accepted"] == n
    zs = [_two_sample_z(x, y, n, n) for x, y in zip(a["measurements"], b["measurements"])]
    assert len(zs) == 22 and max(zs) < 5.0, zs


# ---------------------------------------------------------------------------- config 4
@pytest.mark.parametrize("flags", [FS_RNG_SPLITMIX | FS_FORCE_SEGMENTED, FS_RNG_PHILOX | FS_FORCE_SEGMENTED,
                                   FS_RNG_SPLITMIX])
def test_gpu_config4_deep_trace_matches_reference(cuda, flags):
    """Accepted trajectories reach k_max = 12: the segmented engine's warp / CTA-per-shot block
    kernels (and the general interpreter) against reference amplitudes at k = 10-12."""
    g = load_deep("config4_deep")
    P = g["prog"]
    dp = _dev(P)
    cps = g["sk_index"].tolist()
    out, tb = _trace_all(dp, g, flags, checkpoints=[c + 1 for c in cps])
    _check_final(P, g, out, tb)
    for j, c in enumerate(cps):
        cp = tb.checkpoint(j)
        assert cp["valid"].all() and cp["k"] >= 10
        np.testing.assert_array_equal(cp["frame_x"], g[f"sk{c}_fx"])
        assert rel_err(cp["gamma"], g[f"sk{c}_gamma"]) < TOL
        check_sketch(cp["amps"], g, c, cp["valid"])


def test_gpu_config4_segmented_trace_checkpoints_every_golden(cuda):
    """The config4 golden's boosted-fault trace shots (most halt early) through the segmented
    engine: halted shots freeze at their PostSelect, checkpoints only for shots still running."""
    g = load("config4")
    P = g["prog"]
    dp = _dev(P)
    cps = g["cp_index"].tolist()
    out, tb = _trace_all(dp, g, FS_RNG_SPLITMIX | FS_FORCE_SEGMENTED, checkpoints=[c + 1 for c in cps])
    np.testing.assert_array_equal(out.measurements(), g["t_meas"])
    np.testing.assert_array_equal(out.detectors(), g["t_det"])
    np.testing.assert_array_equal(out.accepted_bits(), g["t_acc"])
    np.testing.assert_array_equal(tb.frame_x[:, :P.n], g["t_fx"])
    assert rel_err(tb.gamma_c(), g["t_gamma"]) < TOL
    for j, c in enumerate(cps):
        cp = tb.checkpoint(j)
        ok = ~np.isnan(g[f"cp{c}_gamma"])
        np.testing.assert_array_equal(cp["valid"], ok)
        np.testing.assert_array_equal(cp["frame_x"][ok], g[f"cp{c}_fx"][ok])
        assert rel_err(cp["gamma"][ok], g[f"cp{c}_gamma"][ok]) < TOL
        assert rel_err(cp["amps"][ok], g[f"cp{c}_amps"][ok]) < TOL


def test_gpu_config4_philox_matches_oracle_deep(cuda):
    """131,072 shots so that thousands reach the k = 10-12 segments (block kernels)."""
    P = load("config4")["prog"]
    dp = _dev(P)
    n = 131_072
    _, gout, _ = dp.sample_host(n, seed=31, shot0=32 * 9, flags=FS_RNG_PHILOX)
    _, oout, _ = oracle.sample(P, n, seed=31, shot0=32 * 9, flags=FS_RNG_PHILOX)
    np.testing.assert_array_equal(gout.measurements(), oout.measurements())
    np.testing.assert_array_equal(gout.detectors(), oout.detectors())
    np.testing.assert_array_equal(gout.accepted_bits(), oout.accepted_bits())
    counts = dp.segment_counts()  # shots entering each post-select segment
    ops = P.instrs[:, 0] & 0xFF
    bounds = [0] + [i + 1 for i in range(P.num_instrs) if ops[i] == 14 and i + 1 < P.num_instrs] + [P.num_instrs]
    first_deep = next(s for s in range(len(bounds) - 1) if max(P.schedule[bounds[s]:bounds[s + 1]]) >= 10)
    assert counts[first_deep] >= 2000, (first_deep, counts)  # shots that ran k >= 10 block-kernel segments


# ---------------------------------------------------------------------------- acceptance 3
@pytest.mark.parametrize("flags", [FS_RNG_SPLITMIX, FS_RNG_PHILOX, FS_RNG_SPLITMIX | FS_FORCE_HBM])
def test_gpu_acceptance_trajectories_match_reference(cuda, flags):
    for i, d in enumerate(load_accept()):
        P = d["prog"]
        dp = _dev(P)
        m = d["modes"]
        st, out, tb = dp.sample_host(1, seed=int(d["seed"][0]), flags=flags,
                                     fault_modes=None if m.size == 0 else m[None, :],
                                     forced=d["forced"][None, :], want_state=True)
        assert st == 0, i
        np.testing.assert_array_equal(out.measurements()[0], d["meas"])
        np.testing.assert_array_equal(out.detectors()[0], d["det"])
        np.testing.assert_array_equal(out.observables()[0], d["obs"])
        np.testing.assert_array_equal(tb.records[0, :P.record_count], d["rec"])
        np.testing.assert_array_equal(tb.frame_x[0, :P.n], d["fx"])
        assert rel_err(tb.gamma_c()[:1], d["gamma"]) < TOL
        assert rel_err(tb.amps_c()[0], d["amps"]) < TOL
        dp.close()


# ---------------------------------------------------------------------------- renormalize=False
@pytest.mark.parametrize("name", renorm_names())
@pytest.mark.parametrize("engine_flag", [0, FS_FORCE_HBM])
def test_gpu_renormalize_false_matches_reference(cuda, name, engine_flag):
    g = load_renorm(name)
    P = g["prog"]
    dp = _dev(P)
    n = g["f_meas"].shape[0]
    st, out, _ = dp.sample_host(n, seed=int(g["f_seed"][0]), flags=FS_RNG_SPLITMIX | FS_NO_RENORM | engine_flag)
    assert st == 0
    np.testing.assert_array_equal(out.measurements(), g["f_meas"])
    np.testing.assert_array_equal(out.detectors(), g["f_det"])
    np.testing.assert_array_equal(out.accepted_bits(), g["f_acc"])
    ns = g["s_gamma"].shape[0]
    st, out, tb = dp.sample_host(ns, seed=int(g["s_seed"][0]), flags=FS_RNG_SPLITMIX | FS_NO_RENORM | engine_flag,
                                 want_state=True)
    assert st == 0
    assert rel_err(tb.gamma_c(), g["s_gamma"]) < TOL
    total = np.abs(tb.gamma_c()) ** 2 * np.linalg.norm(tb.amps_c(), axis=1) ** 2
    np.testing.assert_allclose(total, g["s_total"], rtol=TOL, atol=0)
    np.testing.assert_array_equal(tb.records[:, :P.record_count], g["s_rec"])
    if "s_amps" in g:
        assert rel_err(tb.amps_c(), g["s_amps"]) < TOL


def test_gpu_renormalize_false_philox_matches_oracle(cuda):
    for name in renorm_names():
        P = load_renorm(name)["prog"]
        dp = _dev(P)
        _, a, _ = dp.sample_host(4096, seed=4, flags=FS_RNG_PHILOX | FS_NO_RENORM)
        _, b, _ = oracle.sample(P, 4096, seed=4, flags=FS_RNG_PHILOX | FS_NO_RENORM)
        np.testing.assert_array_equal(a.measurements(), b.measurements())
        np.testing.assert_array_equal(a.accepted_bits(), b.accepted_bits())


# ---------------------------------------------------------------------------- records / trace API
@pytest.mark.parametrize("name", [c for c in case_names() if "t_rec" in load(c) or "t_modes" in load(c)][:40])
def test_gpu_trace_records_include_hidden(cuda, name):
    """ShotState.records (user + hidden) from the trace outputs == the oracle's (and the
    reference's where the fixture stores them)."""
    g = load(name)
    P = g["prog"]
    if P.k_max >= 16:
        pytest.skip("large-k: covered by the config-3 deep trace")
    dp = _dev(P)
    out, tb = _trace_all(dp, g, FS_RNG_SPLITMIX)
    n = g["t_modes"].shape[0]
    _, _, ob = oracle.sample(P, n, seed=int(g["t_seed"][0]), flags=FS_RNG_SPLITMIX, fault_modes=g["t_modes"],
                             forced=g["t_forced"], want_state=True)
    np.testing.assert_array_equal(tb.records[:, :P.record_count], ob.records[:, :P.record_count])
    if "t_rec" in g:
        np.testing.assert_array_equal(tb.records[:, :P.record_count], g["t_rec"])


@pytest.mark.parametrize("name", [c for c in case_names("toy") + case_names("rand") if "cp_index" in load(c)])
def test_gpu_run_shot_trace_states_match_reference_checkpoints(cuda, name):
    """runtime.run_shot(trace=) (one checkpointed device call): the states its callback sees at the
    fixture's checkpoints equal the reference's trace states."""
    from paper_2604_27058_b200 import runtime as R

    g = load(name)
    P = g["prog"]
    cps = set(g["cp_index"].tolist())
    for s in range(g["t_modes"].shape[0]):
        if not g["t_acc"][s]:
            continue
        fo = {r: int(v) for r, v in enumerate(g["t_forced"][s]) if v >= 0}
        seen = {}

        def tr(state, ins, _i=[0]):
            if _i[0] in cps:
                seen[_i[0]] = (state.frame_x.copy(), complex(state.gamma), state.active_view().copy(), state.k)
            _i[0] += 1

        st = R.ShotState(P, seed=int(g["t_seed"][0]))
        R.run_shot(P, st, shot=s, forced_faults=g["t_modes"][s], forced_outcomes=fo, trace=tr)
        for c in cps:
            fx, gm, amps, k = seen[c]
            np.testing.assert_array_equal(fx, g[f"cp{c}_fx"][s])
            assert abs(gm - g[f"cp{c}_gamma"][s]) <= TOL * max(1.0, abs(g[f"cp{c}_gamma"][s]))
            assert rel_err(amps, g[f"cp{c}_amps"][s]) < TOL
            assert k == int(P.schedule[c])


# ---------------------------------------------------------------------------- NaN
def _nan_program(P):
    """Expand phases replaced by NaN (reference test_runtime.py:274-281)."""
    import dataclasses

    fp = P.fparams.copy()
    Q = P
    hit = False
    for i in range(Q.num_instrs):
        if int(Q.instrs[i, 0]) & 0xFF == 2:  # Expand: w5 = offset of its 8 phase doubles
            off = int(Q.instrs[i, 5])
            fp[off:off + 8] = np.nan
            hit = True
    assert hit
    return dataclasses.replace(P, fparams=fp)


@pytest.mark.parametrize("name,flags", [
    ("toy_htm", FS_RNG_SPLITMIX),                       # general interpreter
    ("toy_htm", FS_RNG_PHILOX),                         # general JIT (NVRTC)
    ("toy_htm", FS_RNG_PHILOX | FS_NO_JIT),             # general interpreter, Philox
    ("toy_htm", FS_RNG_SPLITMIX | FS_FORCE_HBM),        # large-k engine, per-instruction kernels
    ("config2", FS_RNG_PHILOX),                         # general JIT with noise
    ("toy_postselect", FS_RNG_PHILOX),                  # segmented, lane-per-shot
    ("config4", FS_RNG_PHILOX),                         # segmented + block kernels
    ("config4", FS_RNG_SPLITMIX),
    ("fusedk00", FS_RNG_SPLITMIX | FS_FORCE_HBM),      # fused tile passes
])
def test_gpu_nan_raises_shot_error(cuda, name, flags, monkeypatch):
    from paper_2604_27058_b200.engine import ShotError

    if "fusedk" in name:
        monkeypatch.setenv("FS_HBM_FUSED", "1")
    Q = _nan_program(load(name)["prog"])
    dp = _dev(Q)
    n = 4096 if Q.k_max < 12 else 64
    with pytest.raises(ShotError, match="NaN"):
        dp.sample_host(n, seed=1, flags=flags)
    with pytest.raises(ShotError, match="NaN"):
        dp.accumulate(n, seed=1, flags=flags)


def test_gpu_nan_raises_through_run_shot(cuda):
    from paper_2604_27058_b200 import runtime as R

    Q = _nan_program(load("toy_htm")["prog"])
    with pytest.raises(R.ShotError, match="NaN"):
        R.run_shot(Q, shot=0)
    with pytest.raises(R.ShotError, match="NaN"):
        R.sample_accumulate(Q, 1000, seed=0)


# ---------------------------------------------------------------------------- independent references

@pytest.mark.parametrize("name", frameref_names())
@pytest.mark.parametrize("flags,n", [(FS_RNG_PHILOX, 10_000_000), (FS_RNG_SPLITMIX, 1_000_000)])
def test_gpu_rates_match_reference_frame_sampler(cuda, name, flags, n):
    """Detector / observable rates of the engine (the bench's affine kernel for Philox) vs the
    reference's independent Pauli-frame sampler (oracle.py:407-516), |z| < 5."""
    g = load_frameref(name)
    dp = _dev(g["prog"])
    acc = dp.accumulate(n, seed=123, flags=flags)
    ns = int(g["shots"][0])
    assert max_two_sample_z(acc["detectors"], g["det_counts"], n, ns) < 5.0
    assert max_two_sample_z(acc["observables"], g["obs_counts"], n, ns) < 5.0


@pytest.mark.parametrize("flags", [FS_RNG_PHILOX, FS_RNG_SPLITMIX])
def test_gpu_fifty_mirrors_are_deterministic(cuda, flags):
    """Acceptance criterion 2 (test_acceptance.py:110-128): 50 exact U U^dagger circuits x 10^4
    shots, every record 0."""
    for i, P in enumerate(load_mirrors50()):
        acc = _dev(P).accumulate(10_000, seed=i, flags=flags)
        assert not acc["measurements"].any(), i


# ---------------------------------------------------------------------------- block engines
_PSEL = [c for c in case_names() if load(c)["prog"].has_postselect and "t_modes" in load(c)]


@pytest.mark.parametrize("name", _PSEL)
@pytest.mark.parametrize("env", [{"FS_BLOCK_K": "1"}, {"FS_BLOCK_K": "11"}, {}, {"FS_BLOCK_NO_FUSE": "1"},
                                 {"FS_BLOCK_K": "1", "FS_BLOCK_NO_FUSE": "1"}, {"FS_BLOCK_NO_WJIT": "1"},
                                 {"FS_BLOCK_K": "1", "FS_BLOCK_NO_WJIT": "1"}, {"FS_SEG_NO_LJIT": "1"},
                                 {"FS_BLOCK_K": "11", "FS_SEG_NO_LJIT": "1"}])
def test_gpu_block_engines_match_reference_and_oracle(cuda, name, env, monkeypatch):
    """Post-selected programs with every segment through the block engine (FS_BLOCK_K=1: warp or
    CTA per shot from k = 1), through lane-per-shot segments up to k = 10 (FS_BLOCK_K=11), and by
    default: trace against the reference (records, frames, gamma, amplitudes), Philox free
    sampling against the oracle."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    g = load(name)
    P = g["prog"]
    dp = _dev(P)
    out, tb = _trace_all(dp, g, FS_RNG_SPLITMIX | FS_FORCE_SEGMENTED)
    np.testing.assert_array_equal(out.measurements(), g["t_meas"])
    np.testing.assert_array_equal(out.detectors(), g["t_det"])
    np.testing.assert_array_equal(out.accepted_bits(), g["t_acc"])
    np.testing.assert_array_equal(tb.frame_x[:, :P.n], g["t_fx"])
    assert rel_err(tb.gamma_c(), g["t_gamma"]) < TOL
    if "t_amps" in g and g["t_acc"].all():
        assert rel_err(tb.amps_c(), g["t_amps"]) < TOL
    n = 8192
    _, a, _ = dp.sample_host(n, seed=41, shot0=32 * 3, flags=FS_RNG_PHILOX)
    _, b, _ = oracle.sample(P, n, seed=41, shot0=32 * 3, flags=FS_RNG_PHILOX)
    np.testing.assert_array_equal(a.measurements(), b.measurements())
    np.testing.assert_array_equal(a.detectors(), b.detectors())
    np.testing.assert_array_equal(a.accepted_bits(), b.accepted_bits())


# ---------------------------------------------------------------------------- star groups
@pytest.mark.parametrize("k,seed", [(2, 0), (3, 1), (4, 2), (5, 3), (6, 4), (7, 5), (8, 6), (9, 7), (10, 8), (10, 9),
                                    (11, 10), (12, 11)])
@pytest.mark.parametrize("env", [{"FS_BLOCK_K": "1"}, {"FS_BLOCK_K": "1", "FS_BLOCK_NO_JIT": "1"},
                                 {"FS_BLOCK_K": "1", "FS_BLOCK_NO_WJIT": "1"},
                                 {"FS_BLOCK_K": "1", "FS_BLOCK_NO_FUSE": "1"}, {}, {"FS_SEG_NO_LJIT": "1"}])
def test_gpu_star_groups_match_oracle(cuda, k, seed, env, monkeypatch):
    """The block engine's fused ArrayGate runs (star groups: CX / CZ / S through one pivot axis,
    an optional H and ArrayRot, FrameGates in between; interpreter, specialised CTA-per-shot
    kernels in the shared-VM and the packed-frame (fs_wseg.cuh) form, packed-frame warp-per-shot kernels) against the oracle's one-sweep-per-instruction VM on hand-built
    programs (tests/synth.py): records of Philox free sampling bit for bit, and the frame, gamma
    and amplitudes at checkpoints between the runs (the reference stream, trace mode)."""
    from synth import star_program

    for kk, v in env.items():
        monkeypatch.setenv(kk, v)
    P = star_program(k, seed)
    dp = _dev(P)
    n = 2048 if k <= 10 else 256
    _, a, _ = dp.sample_host(n, seed=7, flags=FS_RNG_PHILOX)
    _, b, _ = oracle.sample(P, n, seed=7, flags=FS_RNG_PHILOX)
    np.testing.assert_array_equal(a.measurements(), b.measurements())
    np.testing.assert_array_equal(a.accepted_bits(), b.accepted_bits())
    assert a.accepted_bits().all()
    # the specialised segment kernel compiled (a failed compile would fall back to the interpreter)
    if "FS_BLOCK_K" in env:
        interpreted = "FS_BLOCK_NO_JIT" in env or (k <= 10 and "FS_BLOCK_NO_WJIT" in env)
        assert ("segments: ready kernels=1 " in dp.jit_status()) == (not interpreted), dp.jit_status()
    elif k < 9:  # default threshold: both segments are lane-per-shot (fs_lseg.cuh, FrameGates with SWAP gate by gate)
        assert ("segments: ready kernels=0 lane=2" in dp.jit_status()) == ("FS_SEG_NO_LJIT" not in env), dp.jit_status()
    cuts = P.meta["cuts"]
    ns = 8
    _, g, tb = dp.sample_host(ns, seed=11, flags=FS_RNG_SPLITMIX | FS_FORCE_SEGMENTED, want_state=True,
                              checkpoints=cuts)
    _, o, _ = oracle.sample(P, ns, seed=11, flags=FS_RNG_SPLITMIX)
    np.testing.assert_array_equal(g.measurements(), o.measurements())
    for j, c in enumerate(cuts):
        cp = tb.checkpoint(j)
        _, _, ob = oracle.sample(P, ns, seed=11, flags=FS_RNG_SPLITMIX, stop=c, want_state=True)
        assert cp["valid"].all()
        np.testing.assert_array_equal(cp["frame_x"], ob.frame_x[:, :P.n])
        np.testing.assert_array_equal(cp["frame_z"], ob.frame_z[:, :P.n])
        assert rel_err(cp["gamma"], ob.gamma_c()) < TOL
        assert rel_err(cp["amps"], ob.amps_c()) < TOL
