"""GPU parity: the CUDA engines (through the C ABI) against the reference goldens and the oracle.

* trace mode (all random choices supplied): records / detectors / observables /
  accepted / frames bit-exact vs the REFERENCE; gamma and active amplitudes
  within 1e-10 relative (complex128, north_star);
* free sampling with the reference stream (FS_RNG_SPLITMIX): bit-exact vs the
  reference's own ``sample()`` output;
* free sampling with the Philox stream: bit-exact vs the oracle's restatement
  of that stream; frame engine == general engine on frame-only programs.
"""
from __future__ import annotations

import numpy as np
import pytest

import oracle
from goldens import case_names, load, rel_err
from paper_2604_27058_b200._abi import FS_FORCE_GENERAL, FS_FORCE_HBM, FS_NO_JIT, FS_RNG_PHILOX, FS_RNG_SPLITMIX

pytestmark = pytest.mark.gpu
ALL = case_names()
# programs whose active array lives in HBM (k_max >= 16) go through the large-k engine tests
CASES = [c for c in ALL if load(c)["prog"].k_max < 16]
AMP_TOL = 1e-10


def _dev(P):
    from paper_2604_27058_b200.engine import DeviceProgram

    return DeviceProgram(P)


def _same(a, b):
    np.testing.assert_array_equal(a.measurements(), b.measurements())
    np.testing.assert_array_equal(a.detectors(), b.detectors())
    np.testing.assert_array_equal(a.observables(), b.observables())
    np.testing.assert_array_equal(a.accepted_bits(), b.accepted_bits())


@pytest.mark.parametrize("name", [c for c in ALL if "t_modes" in load(c)])
@pytest.mark.parametrize("flags", [FS_RNG_SPLITMIX, FS_RNG_PHILOX, FS_RNG_SPLITMIX | FS_FORCE_HBM])
def test_gpu_trace_matches_reference(cuda, name, flags):
    g = load(name)
    P = g["prog"]
    dp = _dev(P)
    n = g["t_modes"].shape[0]
    st, out, tb = dp.sample_host(n, seed=int(g["t_seed"][0]), flags=flags, fault_modes=g["t_modes"],
                                 forced=g["t_forced"], want_state=True)
    assert st == 0
    np.testing.assert_array_equal(out.measurements(), g["t_meas"])
    np.testing.assert_array_equal(out.detectors(), g["t_det"])
    np.testing.assert_array_equal(out.observables(), g["t_obs"])
    np.testing.assert_array_equal(out.accepted_bits(), g["t_acc"])
    np.testing.assert_array_equal(tb.frame_x[:, :P.n], g["t_fx"])
    np.testing.assert_array_equal(tb.frame_z[:, :P.n], g["t_fz"])
    assert rel_err(tb.gamma_c(), g["t_gamma"]) < AMP_TOL
    if "t_amps" in g and g["t_acc"].all():
        assert rel_err(tb.amps_c(), g["t_amps"]) < AMP_TOL
    if flags & FS_RNG_SPLITMIX:
        np.testing.assert_array_equal(tb.draws, g["t_draws"])


@pytest.mark.parametrize("name", [c for c in CASES if "t_modes" in load(c) and load(c)["prog"].k_max == 0])
def test_gpu_frame_engine_trace_matches_reference(cuda, name):
    """Frame-only programs through the bit-sliced frame engine (no state outputs requested)."""
    g = load(name)
    P = g["prog"]
    dp = _dev(P)
    assert dp.engine(FS_RNG_PHILOX) == "frame"
    n = g["t_modes"].shape[0]
    st, out, tb = dp.sample_host(n, seed=int(g["t_seed"][0]), flags=FS_RNG_PHILOX,
                                 fault_modes=g["t_modes"], forced=g["t_forced"])
    assert st == 0
    np.testing.assert_array_equal(out.measurements(), g["t_meas"])
    np.testing.assert_array_equal(out.detectors(), g["t_det"])
    np.testing.assert_array_equal(out.observables(), g["t_obs"])
    np.testing.assert_array_equal(out.accepted_bits(), g["t_acc"])


@pytest.mark.parametrize("name", [c for c in CASES if "cp_index" in load(c)])
@pytest.mark.parametrize("engine_flag", [0, FS_FORCE_HBM])
def test_gpu_checkpoints_match_reference(cuda, name, engine_flag):
    g = load(name)
    P = g["prog"]
    dp = _dev(P)
    n = g["t_modes"].shape[0]
    for c in g["cp_index"].tolist():
        st, out, tb = dp.sample_host(n, seed=int(g["t_seed"][0]), flags=FS_RNG_SPLITMIX | engine_flag,
                                     fault_modes=g["t_modes"], forced=g["t_forced"], stop=c + 1,
                                     want_state=True)
        ok = ~np.isnan(g[f"cp{c}_gamma"])
        np.testing.assert_array_equal(tb.frame_x[ok, :P.n], g[f"cp{c}_fx"][ok])
        np.testing.assert_array_equal(tb.frame_z[ok, :P.n], g[f"cp{c}_fz"][ok])
        assert rel_err(tb.gamma_c()[ok], g[f"cp{c}_gamma"][ok]) < AMP_TOL
        assert rel_err(tb.amps_c()[ok], g[f"cp{c}_amps"][ok]) < AMP_TOL


@pytest.mark.parametrize("name", [c for c in CASES if "f_meas" in load(c)])
@pytest.mark.parametrize("engine_flag", [0, FS_FORCE_HBM])
def test_gpu_free_reference_stream_matches_reference(cuda, name, engine_flag):
    g = load(name)
    P = g["prog"]
    dp = _dev(P)
    n = g["f_meas"].shape[0]
    st, out, _ = dp.sample_host(n, seed=int(g["f_seed"][0]), flags=FS_RNG_SPLITMIX | engine_flag)
    assert st == 0
    np.testing.assert_array_equal(out.measurements(), g["f_meas"])
    np.testing.assert_array_equal(out.detectors(), g["f_det"])
    np.testing.assert_array_equal(out.observables(), g["f_obs"])
    np.testing.assert_array_equal(out.accepted_bits(), g["f_acc"])


@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("engine_flag", [0, FS_FORCE_HBM])
def test_gpu_free_philox_matches_oracle(cuda, name, engine_flag):
    P = load(name)["prog"]
    n = 2048 if P.k_max < 12 else 256
    dp = _dev(P)
    _, gout, _ = dp.sample_host(n, seed=77, shot0=64, flags=FS_RNG_PHILOX | engine_flag)
    _, oout, _ = oracle.sample(P, n, seed=77, shot0=64, flags=FS_RNG_PHILOX)
    _same(gout, oout)


@pytest.mark.parametrize("name", [c for c in CASES if load(c)["prog"].k_max == 0])
def test_gpu_frame_engine_equals_general_engine(cuda, name):
    P = load(name)["prog"]
    dp = _dev(P)
    n = 5000
    _, a, _ = dp.sample_host(n, seed=5, flags=FS_RNG_PHILOX)
    _, b, _ = dp.sample_host(n, seed=5, flags=FS_RNG_PHILOX | FS_FORCE_GENERAL)
    _same(a, b)


def test_gpu_accumulate_matches_samples(cuda):
    P = load("config2")["prog"] if "config2" in CASES else load("toy_repetition")["prog"]
    dp = _dev(P)
    n = 100_000
    acc = dp.accumulate(n, seed=9)
    _, out, _ = dp.sample_host(n, seed=9)
    a = out.accepted_bits().astype(bool)
    assert acc["accepted"] == int(a.sum())
    np.testing.assert_array_equal(acc["measurements"], out.measurements()[a].sum(0))
    np.testing.assert_array_equal(acc["detectors"], out.detectors()[a].sum(0))
    np.testing.assert_array_equal(acc["observables"], out.observables()[a].sum(0))


def test_gpu_large_k_config3_philox_matches_oracle(cuda):
    """Config 3 (k = 22, HBM engine) free sampling vs the oracle restatement, 2 shots."""
    P = load("config3")["prog"]
    dp = _dev(P)
    assert dp.engine(0) == "hbm"
    _, gout, _ = dp.sample_host(2, seed=3, flags=FS_RNG_PHILOX)
    _, oout, _ = oracle.sample(P, 2, seed=3, flags=FS_RNG_PHILOX)
    _same(gout, oout)


@pytest.mark.parametrize("name", [c for c in CASES if load(c)["prog"].k_max == 0])
def test_gpu_jit_equals_interpreter(cuda, name, monkeypatch):
    """Affine frame kernel == fault-list frame kernel (NVRTC) == frame interpreter, bit for bit."""
    P = load(name)["prog"]
    dp = _dev(P)
    n = 70_000
    _, a, _ = dp.sample_host(n, seed=11, shot0=32 * 7, flags=FS_RNG_PHILOX)
    assert "affine: ready" in dp.jit_status(), dp.jit_status()
    monkeypatch.setenv("FS_NO_AFFINE", "1")  # switches are read when a program handle is created
    dp2 = _dev(P)
    monkeypatch.delenv("FS_NO_AFFINE")
    _, b, _ = dp2.sample_host(n, seed=11, shot0=32 * 7, flags=FS_RNG_PHILOX)
    assert dp2.jit_status().startswith("ready"), dp2.jit_status()
    _, c, _ = dp.sample_host(n, seed=11, shot0=32 * 7, flags=FS_RNG_PHILOX | FS_NO_JIT)
    _same(a, c)
    _same(b, c)


@pytest.mark.parametrize("name", ["config1", "aff_mixed", "aff_rep_psel", "toy_certain", "rand06", "aff_surface_d7",
                                  "aff_many_coins"])
@pytest.mark.parametrize("env", [{}, {"FS_AFF_GLOBAL_TABLES": "1"}, {"FS_AFF_PAIRS": "1"}, {"FS_AFF_NONUNIFORM": "1"},
                                 {"FS_AFF_NO_DIFF": "1"}, {"FS_AFF_PARENTS": "1"}, {"FS_AFF_ANY_PARENTS": "1"},
                                 {"FS_AFF_BALANCED": "1"}, {"FS_AFF_CLS_TABLES": "1"}, {"FS_AFF_DET_PARENTS": "1"},
                                 {"FS_AFF_PAIRS": "16"}, {"FS_AFF_NO_SAFEZONE": "1"}])
@pytest.mark.parametrize("n", [3 * 256 + 37, 3 * 256 + 69])  # even / odd output stride (26 / 27 words)
def test_gpu_affine_variants_match_oracle(cuda, name, env, n, monkeypatch):
    """Affine frame kernel variants (fault tables in global memory, one warp pair per block, the
    exact-bisect case pick, no / single-parent / detector-only / any-row differencing, load-balanced
    row loop, class parameters from tables instead of constants, 16 pairs = named barrier 0, case
    pick always through the cumulative table) == oracle,
    bit for bit; odd shot counts and an offset so the tail word, partial groups and an odd output
    stride are exercised."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    P = load(name)["prog"]
    dp = _dev(P)  # a fresh program handle: the kernel is generated at its first sample call
    _, g, _ = dp.sample_host(n, seed=19, shot0=32 * 5, flags=FS_RNG_PHILOX)
    assert "affine: ready" in dp.jit_status(), dp.jit_status()
    _, o, _ = oracle.sample(P, n, seed=19, shot0=32 * 5, flags=FS_RNG_PHILOX)
    _same(g, o)


@pytest.mark.parametrize("name", [c for c in CASES if 0 < load(c)["prog"].k_max <= 7 and not load(c)["prog"].has_postselect
                                  and not (set((load(c)["prog"].instrs[:, 0] & 0xFF).tolist()) & {7, 9})])
def test_gpu_general_jit_equals_interpreter(cuda, name):
    """Program-specialised general kernel (NVRTC) == general interpreter, bit for bit."""
    P = load(name)["prog"]
    dp = _dev(P)
    n = 20_000
    _, a, _ = dp.sample_host(n, seed=13, shot0=32 * 3, flags=FS_RNG_PHILOX)
    _, b, _ = dp.sample_host(n, seed=13, shot0=32 * 3, flags=FS_RNG_PHILOX | FS_NO_JIT)
    _same(a, b)
    assert dp.jit_status().startswith("ready"), dp.jit_status()


FUSED = [c for c in ALL if load(c)["prog"].k_max >= 12]


def _hbm_plan(dp):
    """(steps, fused passes, fused ops, unfused array kernels, measurements) of the large-k plan."""
    import ctypes as C

    out = (C.c_int64 * 9)()
    dp._lib.fs_debug_hbm_plan.argtypes = [C.c_void_p, C.POINTER(C.c_int64)]
    assert dp._lib.fs_debug_hbm_plan(dp._h, out) == 0
    return list(out)


@pytest.mark.parametrize("name", [c for c in FUSED if "t_modes" in load(c)])
@pytest.mark.parametrize("tma", [False, True])
def test_gpu_fused_passes_trace_match_reference(cuda, name, tma, monkeypatch):
    """Large-k engine with fused tile passes (FS_HBM_FUSED; tiles staged by cp.async or by TMA bulk
    copies) on every k_max >= 12 golden: trace records, frames, gamma, final amplitudes and
    checkpoints against the REFERENCE."""
    monkeypatch.setenv("FS_HBM_FUSED", "1")
    if tma:
        monkeypatch.setenv("FS_PASS_TMA", "1")
    g = load(name)
    P = g["prog"]
    dp = _dev(P)
    assert _hbm_plan(dp)[1] > 0, "no fused pass planned"
    n = g["t_modes"].shape[0]
    flags = FS_RNG_SPLITMIX | FS_FORCE_HBM
    st, out, tb = dp.sample_host(n, seed=int(g["t_seed"][0]), flags=flags, fault_modes=g["t_modes"],
                                 forced=g["t_forced"], want_state=True)
    assert st == 0
    np.testing.assert_array_equal(out.measurements(), g["t_meas"])
    np.testing.assert_array_equal(out.detectors(), g["t_det"])
    np.testing.assert_array_equal(out.accepted_bits(), g["t_acc"])
    np.testing.assert_array_equal(tb.frame_x[:, :P.n], g["t_fx"])
    assert rel_err(tb.gamma_c(), g["t_gamma"]) < AMP_TOL
    if "t_amps" in g and g["t_acc"].all():
        assert rel_err(tb.amps_c(), g["t_amps"]) < AMP_TOL
    for c in (g["cp_index"].tolist() if "cp_index" in g else []):
        st, out, tb = dp.sample_host(n, seed=int(g["t_seed"][0]), flags=flags, fault_modes=g["t_modes"],
                                     forced=g["t_forced"], stop=c + 1, want_state=True)
        ok = ~np.isnan(g[f"cp{c}_gamma"])
        assert rel_err(tb.gamma_c()[ok], g[f"cp{c}_gamma"][ok]) < AMP_TOL
        assert rel_err(tb.amps_c()[ok], g[f"cp{c}_amps"][ok]) < AMP_TOL


@pytest.mark.parametrize("name", [c for c in FUSED if "f_meas" in load(c)])
def test_gpu_fused_passes_free_match_reference(cuda, name, monkeypatch):
    monkeypatch.setenv("FS_HBM_FUSED", "1")
    g = load(name)
    dp = _dev(g["prog"])
    n = g["f_meas"].shape[0]
    st, out, _ = dp.sample_host(n, seed=int(g["f_seed"][0]), flags=FS_RNG_SPLITMIX | FS_FORCE_HBM)
    assert st == 0
    np.testing.assert_array_equal(out.measurements(), g["f_meas"])
    np.testing.assert_array_equal(out.detectors(), g["f_det"])
    np.testing.assert_array_equal(out.accepted_bits(), g["f_acc"])
