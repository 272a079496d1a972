"""Generate golden fixtures from the REFERENCE implementation (run in the build container only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Imports the reference ``framesim`` package from /root/reference (read-only),
compiles circuits with the reference compiler, serializes the programs with
``paper_2604_27058_b200.program.serialize`` and records what the REFERENCE VM
(``framesim.runtime``) produces:

* free sampling with the reference SplitMix64 stream (``sample(prog, S, seed)``):
  measurement / detector / observable bits and ``accepted`` per shot;
* trace mode (SURVEY §8(d) recipe): a per-shot fault plan (2 = off, 3+c = case c,
  drawn with numpy at rate site_prob x boost), the outcomes of every random
  measurement record of a free ``run_shot`` under that plan, then a second
  ``run_shot`` under another seed/shot with both supplied -- its records,
  detectors, observables, accepted flag, frames, gamma and active array (at the
  end and at checkpoints via ``trace``) are stored;
* config programs (BASELINE.json configs 0-4) for bench.py.

Nothing here is imported by the tests: they read the .npz files.
"""
from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")

from framesim.backend import compile_circuit  # noqa: E402  (reference)
from framesim.circuit import parse_circuit  # noqa: E402
from framesim.runtime import ShotState, run_shot, sample  # noqa: E402
from framesim import testing as ftest  # noqa: E402

from paper_2604_27058_b200.configs import CONFIGS, config_text  # noqa: E402
from paper_2604_27058_b200.program import serialize  # noqa: E402

OUT = ROOT / "tests" / "golden"
PROGS = ROOT / "paper_2604_27058_b200" / "programs"
RANDOM_KINDS = ("MeasDormantRandom", "MeasActive", "MeasCollapse")

# irreducible peak dimension 10 (same construction as the reference's performance smoke,
# test_acceptance.py criterion 10): rotation layer, global parity readout, X readouts
_K10 = "\n".join([f"R_Y(0.7) {q}" for q in range(10)] + [f"CX {q} {q + 1}" for q in range(9)]
                 + ["M 9"] + [f"CX {q} {q + 1}" for q in range(8, -1, -1)]
                 + ["MX " + " ".join(str(q) for q in range(10))]) + "\n"


def free_golden(prog, shots, seed):
    recs = list(sample(prog, shots, seed=seed))
    U, D, O = len(prog.user_records), prog.num_detectors, prog.num_observables
    meas = np.array([r.measurements for r in recs], dtype=np.uint8).reshape(shots, U)
    det = np.array([r.detectors for r in recs], dtype=np.uint8).reshape(shots, D)
    obs = np.array([r.observables for r in recs], dtype=np.uint8).reshape(shots, O)
    acc = np.array([r.accepted for r in recs], dtype=np.uint8)
    return meas, det, obs, acc


def trace_golden(prog, shots, seed, boost, rng, checkpoints=()):
    E = len(prog.sites)
    R = prog.record_count
    rand_records = {ins.record for ins in prog.instrs if type(ins).__name__ in RANDOM_KINDS}
    modes = np.full((shots, E), 2, dtype=np.int16)
    forced = np.full((shots, R), -1, dtype=np.int8)
    rows = {k: [] for k in ("meas", "det", "obs", "acc", "fx", "fz", "gamma", "k", "amps", "draws", "rec")}
    cps = {c: {"fx": [], "fz": [], "gamma": [], "amps": []} for c in checkpoints}
    for s in range(shots):
        for site, tab in enumerate(prog.sites):
            if tab.case_cum and rng.random() < min(1.0, tab.prob * boost):
                modes[s, site] = 3 + int(rng.integers(0, len(tab.case_cum)))
        st = ShotState(prog, seed=seed + 17)
        run_shot(prog, st, shot=1000 + s, forced_faults=modes[s])
        for r in rand_records:
            forced[s, r] = int(st.records[r])
        snap = {}

        def tr(state, ins, _idx=[0]):
            i = _idx[0]
            _idx[0] += 1
            if i in cps:
                snap[i] = (state.frame_x.copy(), state.frame_z.copy(), complex(state.gamma),
                           state.active_view().copy())

        st2 = ShotState(prog, seed=seed)
        fo = {int(r): int(forced[s, r]) for r in rand_records}
        rec = run_shot(prog, st2, shot=s, forced_faults=modes[s], forced_outcomes=fo,
                       trace=tr if checkpoints else None)
        rows["meas"].append(rec.measurements.astype(np.uint8))
        rows["det"].append(rec.detectors.astype(np.uint8))
        rows["obs"].append(rec.observables.astype(np.uint8))
        rows["acc"].append(int(rec.accepted))
        rows["fx"].append(st2.frame_x.copy())
        rows["fz"].append(st2.frame_z.copy())
        rows["gamma"].append(complex(st2.gamma))
        rows["k"].append(st2.k)
        rows["amps"].append(st2.active_view().copy())
        rows["draws"].append(st2.rng.draws)
        rows["rec"].append(st2.records.copy())
        for c in checkpoints:
            if c in snap:
                fx, fz, g, a = snap[c]
            else:  # shot halted before the checkpoint
                fx = fz = np.zeros(prog.n, np.uint8)
                g, a = complex("nan"), np.full(1 << prog.active_schedule[c], np.nan + 0j)
            cps[c]["fx"].append(fx)
            cps[c]["fz"].append(fz)
            cps[c]["gamma"].append(g)
            cps[c]["amps"].append(a)
    U, D, O = len(prog.user_records), prog.num_detectors, prog.num_observables
    out = {
        "t_modes": modes, "t_forced": forced,
        "t_meas": np.array(rows["meas"], np.uint8).reshape(shots, U),
        "t_det": np.array(rows["det"], np.uint8).reshape(shots, D),
        "t_obs": np.array(rows["obs"], np.uint8).reshape(shots, O),
        "t_acc": np.array(rows["acc"], np.uint8),
        "t_fx": np.array(rows["fx"], np.uint8), "t_fz": np.array(rows["fz"], np.uint8),
        "t_gamma": np.array(rows["gamma"], np.complex128), "t_k": np.array(rows["k"], np.int32),
        "t_draws": np.array(rows["draws"], np.int64),
        "t_rec": np.array(rows["rec"], np.uint8).reshape(shots, R),  # all records, hidden included
    }
    ks = set(rows["k"])
    if len(ks) == 1:  # every shot ends at the same k unless some halted
        out["t_amps"] = np.array(rows["amps"], np.complex128)
    out["t_seed"] = np.array([seed])
    if checkpoints:
        out["cp_index"] = np.array(checkpoints, np.int32)
        for c in checkpoints:
            out[f"cp{c}_fx"] = np.array(cps[c]["fx"], np.uint8)
            out[f"cp{c}_fz"] = np.array(cps[c]["fz"], np.uint8)
            out[f"cp{c}_gamma"] = np.array(cps[c]["gamma"], np.complex128)
            out[f"cp{c}_amps"] = np.array(cps[c]["amps"], np.complex128)
    return out


def write_case(name, prog, text, *, free_shots=256, free_seed=3, trace_shots=16, boost=20.0,
               checkpoints=(), rng=None, meta=None):
    t0 = time.time()
    rng = rng or np.random.default_rng(abs(hash(name)) % (2 ** 32))
    P = serialize(prog, name=name, meta=meta or {})
    payload = {"program": np.frombuffer(P.to_npz_bytes(), dtype=np.uint8),
               "circuit": np.array(text)}
    if free_shots:
        m, d, o, a = free_golden(prog, free_shots, free_seed)
        payload.update(f_meas=m, f_det=d, f_obs=o, f_acc=a, f_seed=np.array([free_seed]))
    if trace_shots:
        payload.update(trace_golden(prog, trace_shots, seed=11, boost=boost, rng=rng,
                                    checkpoints=checkpoints))
    np.savez_compressed(OUT / f"{name}.npz", **payload)
    print(f"{name:28s} k_max={prog.k_max:2d} instrs={len(prog.instrs):4d} "
          f"({time.time() - t0:.1f}s)", flush=True)


# ------------------------------------------------------------------ round-2 fixtures
SKETCH_VECS = 4      # <v_i, a> for v_i ~ CN(0, 1)^(2^k), default_rng(SKETCH_SEED + i)
SKETCH_SEED = 4242
SKETCH_ENTRIES = 1024  # sampled entries, indices default_rng(SKETCH_SEED - 1).choice(2^k, 1024)


def sketch_vectors(k):
    """The fixed complex vectors of the amplitude sketch (the tests regenerate them)."""
    out = []
    for i in range(SKETCH_VECS):
        g = np.random.default_rng(SKETCH_SEED + i)
        out.append(g.standard_normal(1 << k) + 1j * g.standard_normal(1 << k))
    idx = np.sort(np.random.default_rng(SKETCH_SEED - 1).choice(1 << k, size=min(SKETCH_ENTRIES, 1 << k),
                                                                  replace=False))
    return out, idx


def sketch(a, vecs, idx):
    """(sum |a|^2, [<v_i, a>], a[idx]) of one amplitude array."""
    a = np.asarray(a, np.complex128)
    return (float(np.vdot(a, a).real), np.array([np.vdot(v, a) for v in vecs], np.complex128),
            a[idx].copy())


def deep_trace_golden(prog, shots, seed, rng, checkpoints, boost=20.0, forced_builder=None):
    """trace_golden for arrays too large to store: the active array at each checkpoint is kept as a
    sketch (norm, inner products with fixed seeded vectors, sampled entries).  ``forced_builder``
    (shot, modes) -> forced outcomes dict replaces the free-run recipe (post-selected programs)."""
    E = len(prog.sites)
    R = prog.record_count
    rand_records = {ins.record for ins in prog.instrs if type(ins).__name__ in RANDOM_KINDS}
    modes = np.full((shots, E), 2, dtype=np.int16)
    forced = np.full((shots, R), -1, dtype=np.int8)
    sk = {c: sketch_vectors(prog.active_schedule[c]) for c in checkpoints}
    rows = {k: [] for k in ("meas", "det", "obs", "acc", "fx", "fz", "gamma", "k", "amps", "draws", "rec")}
    cps = {c: {"fx": [], "fz": [], "gamma": [], "norm2": [], "ip": [], "vals": []} for c in checkpoints}
    for s in range(shots):
        t0 = time.time()
        if forced_builder is None:
            for site, tab in enumerate(prog.sites):
                if tab.case_cum and rng.random() < min(1.0, tab.prob * boost):
                    modes[s, site] = 3 + int(rng.integers(0, len(tab.case_cum)))
            st = ShotState(prog, seed=seed + 17)
            run_shot(prog, st, shot=1000 + s, forced_faults=modes[s])
            fo = {int(r): int(st.records[r]) for r in rand_records}
        else:
            modes[s], fo = forced_builder(s)
        for r, b in fo.items():
            forced[s, r] = b
        snap = {}

        def tr(state, ins, _idx=[0]):
            i = _idx[0]
            _idx[0] += 1
            if i in cps:
                vecs, idx = sk[i]
                snap[i] = (state.frame_x.copy(), state.frame_z.copy(), complex(state.gamma),
                           sketch(state.active_view(), vecs, idx))

        st2 = ShotState(prog, seed=seed)
        rec = run_shot(prog, st2, shot=s, forced_faults=modes[s], forced_outcomes=fo, trace=tr)
        rows["meas"].append(rec.measurements.astype(np.uint8))
        rows["det"].append(rec.detectors.astype(np.uint8))
        rows["obs"].append(rec.observables.astype(np.uint8))
        rows["acc"].append(int(rec.accepted))
        rows["fx"].append(st2.frame_x.copy())
        rows["fz"].append(st2.frame_z.copy())
        rows["gamma"].append(complex(st2.gamma))
        rows["k"].append(st2.k)
        rows["amps"].append(st2.active_view().copy())
        rows["draws"].append(st2.rng.draws)
        rows["rec"].append(st2.records.copy())
        for c in checkpoints:
            kc = prog.active_schedule[c]
            if c in snap:
                fx, fz, g, (n2, ip, vals) = snap[c]
            else:
                fx = fz = np.zeros(prog.n, np.uint8)
                g, n2 = complex("nan"), float("nan")
                ip = np.full(SKETCH_VECS, np.nan + 0j)
                vals = np.full(min(SKETCH_ENTRIES, 1 << kc), np.nan + 0j)
            cps[c]["fx"].append(fx)
            cps[c]["fz"].append(fz)
            cps[c]["gamma"].append(g)
            cps[c]["norm2"].append(n2)
            cps[c]["ip"].append(ip)
            cps[c]["vals"].append(vals)
        print(f"  shot {s}: accepted={rec.accepted} ({time.time() - t0:.1f}s)", flush=True)
    U, D, O = len(prog.user_records), prog.num_detectors, prog.num_observables
    out = {
        "t_modes": modes, "t_forced": forced,
        "t_meas": np.array(rows["meas"], np.uint8).reshape(shots, U),
        "t_det": np.array(rows["det"], np.uint8).reshape(shots, D),
        "t_obs": np.array(rows["obs"], np.uint8).reshape(shots, O),
        "t_acc": np.array(rows["acc"], np.uint8),
        "t_fx": np.array(rows["fx"], np.uint8), "t_fz": np.array(rows["fz"], np.uint8),
        "t_gamma": np.array(rows["gamma"], np.complex128), "t_k": np.array(rows["k"], np.int32),
        "t_draws": np.array(rows["draws"], np.int64),
        "t_rec": np.array(rows["rec"], np.uint8).reshape(shots, R),
        "t_seed": np.array([seed]),
        "sk_index": np.array(checkpoints, np.int32),
        "sk_seed": np.array([SKETCH_SEED, SKETCH_VECS, SKETCH_ENTRIES]),
    }
    if len(set(rows["k"])) == 1:
        out["t_amps"] = np.array(rows["amps"], np.complex128)
    for c in checkpoints:
        out[f"sk{c}_idx"] = sk[c][1]
        out[f"sk{c}_fx"] = np.array(cps[c]["fx"], np.uint8)
        out[f"sk{c}_fz"] = np.array(cps[c]["fz"], np.uint8)
        out[f"sk{c}_gamma"] = np.array(cps[c]["gamma"], np.complex128)
        out[f"sk{c}_norm2"] = np.array(cps[c]["norm2"], np.float64)
        out[f"sk{c}_ip"] = np.array(cps[c]["ip"], np.complex128)
        out[f"sk{c}_vals"] = np.array(cps[c]["vals"], np.complex128)
    return out


def accepted_forced_builder(prog, text, rng, boost):
    """Forced faults + forced outcomes under which the post-selected program ACCEPTS the shot.

    Pauli-frame updates are GF(2)-affine in the recorded outcomes, so with the faults fixed the
    detector vector is an affine function of the MeasDormantRandom coins: probe it column by
    column on the same circuit compiled WITHOUT post-selection (same records and sites), solve
    detectors = 0 for the coin flips, then confirm on the post-selected program (a forced
    MeasCollapse record that became impossible, or any mismatch, draws a new fault plan)."""
    from framesim.runtime import ShotError

    prog_np = compile_circuit(text)
    assert prog_np.record_count == prog.record_count and len(prog_np.sites) == len(prog.sites)
    E = len(prog.sites)
    rand_records = [ins.record for ins in prog.instrs if type(ins).__name__ in RANDOM_KINDS]
    coins = [ins.record for ins in prog_np.instrs if type(ins).__name__ == "MeasDormantRandom"]
    D = prog.num_detectors

    def dets(modes, fo, seed):
        st = ShotState(prog_np, seed=seed)
        rec = run_shot(prog_np, st, shot=0, forced_faults=modes, forced_outcomes=fo)
        return np.asarray(rec.detectors, np.uint8), st

    def solve(A, b):  # one random solution of A x = b over GF(2), or None
        A = A.copy() % 2
        b = b.copy() % 2
        m, n = A.shape
        piv = []
        r = 0
        for c in rng.permutation(n):
            rows = [i for i in range(r, m) if A[i, c]]
            if not rows:
                continue
            A[[r, rows[0]]] = A[[rows[0], r]]
            b[[r, rows[0]]] = b[[rows[0], r]]
            for i in range(m):
                if i != r and A[i, c]:
                    A[i] ^= A[r]
                    b[i] ^= b[r]
            piv.append((r, c))
            r += 1
            if r == m:
                break
        if any(b[i] for i in range(r, m)):
            return None
        x = np.zeros(n, np.uint8)
        free = [c for c in range(n) if c not in {c for _, c in piv}]
        x[free] = rng.integers(0, 2, len(free))
        for row, c in reversed(piv):
            x[c] = (b[row] + (A[row] @ x) - A[row, c] * x[c]) % 2
        return x

    cache = {}

    def build(s):
        for attempt in range(50):
            modes = np.full(E, 2, dtype=np.int16)
            for site, tab in enumerate(prog.sites):
                if tab.case_cum and rng.random() < min(1.0, tab.prob * boost):
                    modes[site] = 3 + int(rng.integers(0, len(tab.case_cum)))
            seed = 7000 + 101 * s + attempt
            try:
                d0, st = dets(modes, None, seed)
            except ShotError:
                continue
            base = {int(r): int(st.records[r]) for r in rand_records}
            if "A" not in cache:  # coin -> detector columns (fault-plan independent)
                cols = []
                for c in coins:
                    fo = dict(base)
                    fo[c] ^= 1
                    try:
                        dc, _ = dets(modes, fo, seed)
                    except ShotError:
                        dc = None
                    cols.append(np.zeros(D, np.uint8) if dc is None else dc ^ d0)
                cache["A"] = np.array(cols, np.uint8).T
            x = solve(cache["A"], d0)
            if x is None:
                continue
            fo = dict(base)
            for c, f in zip(coins, x):
                fo[c] ^= int(f)
            try:
                st2 = ShotState(prog, seed=seed)
                rec = run_shot(prog, st2, shot=0, forced_faults=modes, forced_outcomes=fo)
            except ShotError:
                continue
            if rec.accepted:
                return modes, fo
        raise RuntimeError("no accepted trajectory found")

    return build


def main(which=("configs", "random", "toys")):
    OUT.mkdir(exist_ok=True)
    (OUT / "deep").mkdir(exist_ok=True)
    PROGS.mkdir(exist_ok=True)
    if "toys" in which:
        toys = {
            "toy_htm": ("H 0\nT 0\nH 0\nM 0\n", {}),
            "toy_noise_twice": ("H 0\nT 0\nH 0\nM 0\nDEPOLARIZE1(0.3) 0\nM 0\n", {}),
            "toy_mirror": ("H 0\nT 0\nT 0\nT 0\nCX 0 1\nCX 0 1\nS_DAG 0\nT_DAG 0\nH 0\nM 0 1\n", {}),
            "toy_worked": ("H 0\nT 0\nT 0\nT 0\nCX 0 1\nDEPOLARIZE1(0.001) 0 1\nCX 0 1\nT_DAG 0\nH 0\nM 0 1\n", {}),
            "toy_postselect": ("H 0\nM 0\nPOSTSELECT rec[-1]\nH 1\nT 1\nH 1\nM 1\nDEPOLARIZE1(0.5) 1\nM 1\n", {}),
            "toy_postselect1": ("H 0\nM 0\nPOSTSELECT(1) rec[-1]\nM 0\n", {}),
            "toy_certain": ("X_ERROR(1.0) 0\nX_ERROR(0.5) 1\nX_ERROR(0.0) 2\nDEPOLARIZE1(1.0) 3\nM 0 1 2 3\n",
                            {"optimize": False}),
            "toy_unopt_active": ("H 0\nT 0\nH 1\nT 1\nCX 0 1\nH 0\nM 0\nH 1\nM 1\nR_X(0.3) 2\nMX 2\n",
                                 {"optimize": False}),
            "toy_feedforward": ("H 0\nT 0\nH 0\nM 0\nCX rec[-1] 1\nX_ERROR(0.3) 1\nM 1\nDETECTOR rec[-1] rec[-2]\n"
                                "OBSERVABLE_INCLUDE(0) rec[-1]\nOBSERVABLE_INCLUDE(0) rec[-2]\n", {}),
            "toy_repetition": (str(ftest.repetition_code_circuit(3, 5, 0.05)), {}),
            "toy_pad200": ("R_Y(0.7) 0\nR_Y(0.7) 1\nCX 0 1\nM 1\nCX 0 1\nMX 0 1\nZ 199\n", {}),
            "toy_k10": (_K10, {}),
            "toy_k10_pad200": (_K10 + "Z 199\n", {}),
        }
        for name, (text, kw) in toys.items():
            prog = compile_circuit(text, optimize=kw.get("optimize", True))
            write_case(name, prog, text, free_shots=512, trace_shots=12,
                       checkpoints=tuple(range(min(len(prog.instrs), 6))))
    if "random" in which:
        rng = np.random.default_rng(20261019)
        for i in range(24):
            n = int(rng.integers(2, 9))
            kw = dict(p_noise=float(rng.choice([0.0, 0.05, 0.3])),
                      measure_rate=float(rng.uniform(0.1, 0.3)),
                      rot_rate=float(rng.uniform(0.1, 0.35)),
                      reset_rate=float(rng.choice([0.0, 0.05])),
                      feedforward_rate=float(rng.choice([0.0, 0.08])),
                      measure_all=bool(rng.random() < 0.6),
                      max_noncliff=int(rng.integers(3, 11)))
            circ = ftest.random_circuit(rng, n, int(rng.integers(8, 40)), **kw)
            text = str(circ)
            opt = bool(rng.random() < 0.8)
            prog = compile_circuit(text, optimize=opt)
            cps = tuple(sorted(set(int(x) for x in rng.integers(0, len(prog.instrs), size=3))))
            write_case(f"rand{i:02d}", prog, text, free_shots=256, trace_shots=10,
                       checkpoints=cps, rng=rng, meta={"optimize": opt, **kw})
        from paper_2604_27058_b200.configs import random_near_clifford
        for i in range(8):  # rotation-heavy: larger active dimension (config-0-like, own sizes)
            n = int(rng.integers(6, 12))
            text = random_near_clifford(n, int(rng.integers(4, 9)), t_cells=int(rng.integers(5, 11)),
                                        seed=int(rng.integers(0, 2 ** 31)))
            lines = text.strip().split("\n")
            if i % 2:  # keep the final active array alive: measure only half the qubits
                lines[-1] = "M " + " ".join(str(q) for q in range(0, n, 2))
            if i % 4 >= 2:  # sprinkle noise
                lines = [x for ln in lines for x in (ln, f"DEPOLARIZE1(0.02) {rng.integers(0, n)}")]
            text = "\n".join(lines) + "\n"
            prog = compile_circuit(text)
            cps = tuple(sorted(set(int(x) for x in rng.integers(0, len(prog.instrs), size=3))))
            write_case(f"bigk{i:02d}", prog, text, free_shots=128, trace_shots=6, checkpoints=cps,
                       rng=rng)
        for i in range(6):
            circ = ftest.random_mirror_circuit(rng, int(rng.integers(2, 7)), int(rng.integers(1, 8)))
            text = str(circ)
            write_case(f"mirror{i:02d}", compile_circuit(text), text, free_shots=512, trace_shots=4, rng=rng)
    if "fused" in which:  # 12 <= k_max <= 15: the large-k engine's fused tile passes at small sizes
        from paper_2604_27058_b200.configs import random_near_clifford
        rng = np.random.default_rng(7)
        made = 0
        while made < 4:
            n = int(rng.integers(13, 18))
            text = random_near_clifford(n, int(rng.integers(4, 9)), t_cells=int(rng.integers(10, 25)),
                                        seed=int(rng.integers(0, 2 ** 31)))
            prog = compile_circuit(text)
            if not 12 <= prog.k_max <= 15:
                continue
            lines = text.strip().split("\n")
            if made % 2:
                lines[-1] = "M " + " ".join(str(q) for q in range(0, n, 2))
            if made >= 2:
                lines = [x for ln in lines for x in (ln, f"DEPOLARIZE1(0.02) {rng.integers(0, n)}")]
            text = "\n".join(lines) + "\n"
            prog = compile_circuit(text)
            cps = tuple(sorted(set(int(x) for x in rng.integers(0, len(prog.instrs), size=3))))
            write_case(f"fusedk{made:02d}", prog, text, free_shots=64, trace_shots=4, checkpoints=cps, rng=rng)
            made += 1
    if "formats" in which:  # reference CLI bytes (cli.py:72-113) for the device output formats
        from framesim import cli as fcli
        import tempfile
        fdir = OUT / "formats"
        fdir.mkdir(exist_ok=True)
        toys_txt = {
            "toy_repetition": (str(ftest.repetition_code_circuit(3, 5, 0.05)), ""),
            "toy_repetition_ps": (str(ftest.repetition_code_circuit(3, 4, 0.08)), "0,2,3"),
            "toy_postselect": ("H 0\nM 0\nPOSTSELECT rec[-1]\nH 1\nT 1\nH 1\nM 1\nDEPOLARIZE1(0.5) 1\nM 1\n", ""),
            "toy_feedforward": ("H 0\nT 0\nH 0\nM 0\nCX rec[-1] 1\nX_ERROR(0.3) 1\nM 1\nDETECTOR rec[-1] rec[-2]\n"
                                "OBSERVABLE_INCLUDE(0) rec[-1]\nOBSERVABLE_INCLUDE(0) rec[-2]\n", ""),
            "toy_worked": ("H 0\nT 0\nT 0\nT 0\nCX 0 1\nDEPOLARIZE1(0.001) 0 1\nCX 0 1\nT_DAG 0\nH 0\nM 0 1\n", ""),
            "surface_d3": (config_text(2)[0], ""),
        }
        for name, (text, ps) in toys_txt.items():
            t0 = time.time()
            pstuple = tuple(int(x) for x in ps.split(",")) if ps else ()
            prog = compile_circuit(text, postselect_detectors=pstuple)
            payload = {"program": np.frombuffer(serialize(prog, name=name).to_npz_bytes(), dtype=np.uint8),
                       "circuit": np.array(text), "postselect": np.array(ps), "shots": np.array([300]),
                       "seed": np.array([7])}
            with tempfile.TemporaryDirectory() as td:
                cpath = f"{td}/c.txt"
                open(cpath, "w").write(text)
                for fmt in ("01", "bin", "csv"):
                    for keep in (False, True):
                        opath = f"{td}/o_{fmt}_{int(keep)}"
                        argv = ["sample", cpath, "--shots", "300", "--seed", "7", "--format", fmt, "--out", opath]
                        if ps:
                            argv += ["--postselect-detectors", ps]
                        if keep:
                            argv.append("--keep-rejected")
                        assert fcli.main(argv) == 0
                        payload[f"{fmt}_{int(keep)}"] = np.frombuffer(open(opath, "rb").read(), dtype=np.uint8)
            np.savez_compressed(fdir / f"{name}.npz", **payload)
            print(f"formats/{name:20s} ({time.time() - t0:.1f}s)", flush=True)
    if "affine" in which:  # frame-only programs exercising the affine frame kernel's paths
        rng_a = np.random.default_rng(77)
        # repetition memory with post-selected early detectors and an observable across them
        rep = []
        d, rounds = 5, 4
        data, anc = list(range(0, 2 * d - 1, 2)), list(range(1, 2 * d - 1, 2))
        for r in range(rounds):
            rep.append("DEPOLARIZE1(0.01) " + " ".join(map(str, data)))
            for a in anc:
                rep.append(f"CX {a - 1} {a}\nCX {a + 1} {a}")
            rep.append("X_ERROR(0.02) " + " ".join(map(str, anc)))
            rep.append("M " + " ".join(map(str, anc)))
            for j in range(len(anc)):
                k = len(anc) - j
                rep.append(f"DETECTOR rec[-{k}]" + (f" rec[-{k + len(anc)}]" if r else ""))
            rep.append("R " + " ".join(map(str, anc)))
        rep.append("X_ERROR(0.02) " + " ".join(map(str, data)))
        rep.append("M " + " ".join(map(str, data)))
        rep.append("OBSERVABLE_INCLUDE(0) rec[-1]")
        # mixed noise: several probabilities (runs), near-equal ones (thinning), certain sites,
        # Y/Z errors, MX/MY, resets, detectors and in-circuit POSTSELECT
        mix = []
        n = 6
        for layer in range(8):
            for q in range(n):
                mix.append(["H", "S", "S_DAG", "X", "Y", "Z"][int(rng_a.integers(6))] + f" {q}")
            perm = rng_a.permutation(n)
            mix.append("CX " + " ".join(str(int(x)) for x in perm))
            mix.append(f"DEPOLARIZE2(0.03) " + " ".join(str(int(x)) for x in perm))
            mix.append(f"Y_ERROR(0.02) {layer % n}\nZ_ERROR(0.02) {(layer + 1) % n}")
            mix.append(f"X_ERROR({0.02 * (1 + 1e-12)!r}) {(layer + 2) % n}")
            if layer == 3:
                mix.append("X_ERROR(1.0) 2\nDEPOLARIZE1(1.0) 4")
            if layer % 2 == 1:
                mix.append(f"MX {layer % n}\nMY {(layer + 3) % n}\nDETECTOR rec[-1] rec[-2]\nR {layer % n} {(layer + 3) % n}")
            if layer == 5:
                mix.append("M 1\nPOSTSELECT rec[-1]")
        mix.append("M " + " ".join(map(str, range(n))))
        mix.append("DETECTOR rec[-1] rec[-2]\nOBSERVABLE_INCLUDE(0) rec[-3] rec[-6]\nOBSERVABLE_INCLUDE(1) rec[-4]")
        from paper_2604_27058_b200.configs import rotated_surface_code
        aff = {
            # a larger frame-only program: ~1000 output rows, ~10^4 fault elements (table sizes,
            # shared-memory budget and launch shape of the affine kernel away from config 1's)
            "aff_surface_d7": (rotated_surface_code(7, 7, 2e-3), ()),
            # > 128 coins: 20 qubits measured in a random basis 12 times (240 random outcomes)
            "aff_many_coins": ("".join(f"H {' '.join(map(str, range(20)))}\nDEPOLARIZE1(0.01) {' '.join(map(str, range(20)))}\n"
                                       f"M {' '.join(map(str, range(20)))}\nDETECTOR rec[-1] rec[-2]\n"
                                       f"R {' '.join(map(str, range(20)))}\n" for _ in range(12))
                               + "OBSERVABLE_INCLUDE(0) rec[-1] rec[-3]\n", ()),
            "aff_rep_psel": ("\n".join(rep) + "\n", (0, 1, 2, 3, 5, 6)),
            "aff_rep": ("\n".join(rep) + "\n", ()),
            "aff_mixed": ("\n".join(mix) + "\n", ()),
        }
        for name, (text, ps) in aff.items():
            prog = compile_circuit(text, optimize=True, postselect_detectors=ps)
            assert prog.k_max == 0, name
            write_case(name, prog, text, free_shots=512, trace_shots=16, boost=5.0)
    if "stratum" in which:  # stratified importance sampling (runtime.py:886-945)
        from framesim.runtime import StratumSpec
        from framesim import cli as fcli
        import tempfile
        sdir = OUT / "stratum"
        sdir.mkdir(exist_ok=True)
        from paper_2604_27058_b200.configs import random_near_clifford
        nc_text = random_near_clifford(6, 5, t_cells=6, seed=11)
        nc_lines = nc_text.strip().split("\n")
        nc_lines = [x for ln in nc_lines for x in (ln, "DEPOLARIZE1(0.02) 1 3")]
        cases = {
            "repetition": (str(ftest.repetition_code_circuit(3, 5, 0.05)), True, ()),
            "postselect": ("H 0\nM 0\nPOSTSELECT rec[-1]\nH 1\nT 1\nH 1\nM 1\nDEPOLARIZE1(0.5) 1\nM 1\n", True, ()),
            "noise_twice": ("H 0\nT 0\nH 0\nM 0\nDEPOLARIZE1(0.3) 0\nM 0\n", True, ()),
            "certain": ("X_ERROR(1.0) 0\nX_ERROR(0.5) 1\nX_ERROR(0.0) 2\nDEPOLARIZE1(1.0) 3\nM 0 1 2 3\n", False, ()),
            "surface_d3": (config_text(2)[0], True, ()),
            "near_clifford": ("\n".join(nc_lines) + "\n", True, ()),
            "repetition_ps": (str(ftest.repetition_code_circuit(3, 4, 0.08)), True, (0, 2, 3)),
        }
        for name, (text, opt, ps) in cases.items():
            t0 = time.time()
            prog = compile_circuit(text, optimize=opt, postselect_detectors=ps)
            E = len(prog.sites)
            payload = {"program": np.frombuffer(serialize(prog, name=name).to_npz_bytes(), dtype=np.uint8),
                       "circuit": np.array(text)}
            ws = [w for w in (0, 1, 2, 3, 5) if w <= E]
            payload["ws"] = np.array(ws)
            for w in ws:
                spec = StratumSpec(prog, w)
                recs = list(sample(prog, 96, seed=5, stratum=spec))
                payload[f"w{w}_meas"] = np.array([r.measurements for r in recs], np.uint8).reshape(len(recs), -1)
                payload[f"w{w}_det"] = np.array([r.detectors for r in recs], np.uint8).reshape(len(recs), -1)
                payload[f"w{w}_obs"] = np.array([r.observables for r in recs], np.uint8).reshape(len(recs), -1)
                payload[f"w{w}_acc"] = np.array([r.accepted for r in recs], np.uint8)
                payload[f"w{w}_weight"] = np.array([spec.weight])
                assert all(r.weight == spec.weight for r in recs)
            try:
                StratumSpec(prog, E + 1)
            except ValueError as exc:
                payload["too_many_error"] = np.array(str(exc))
            if opt and not ps:  # the CLI path (compile with defaults) pins the csv weight text
                with tempfile.TemporaryDirectory() as td:
                    cpath, opath = f"{td}/c.txt", f"{td}/o.csv"
                    open(cpath, "w").write(text)
                    w = ws[min(1, len(ws) - 1)]
                    assert fcli.main(["sample", cpath, "--shots", "96", "--seed", "5", "--format", "csv",
                                      "--stratum-w", str(w), "--out", opath, "--keep-rejected"]) == 0
                    payload["cli_w"] = np.array([w])
                    payload["cli_csv"] = np.frombuffer(open(opath, "rb").read(), dtype=np.uint8)
            np.savez_compressed(sdir / f"{name}.npz", **payload)
            print(f"stratum/{name:16s} E={E:4d} ws={ws} ({time.time() - t0:.1f}s)", flush=True)
    if "laws" in which:  # known-answer laws of the reference tests (test_runtime.py, test_acceptance.py)
        ldir = OUT / "laws"
        ldir.mkdir(exist_ok=True)
        laws = {
            "htm": "H 0\nT 0\nH 0\nM 0\n",                     # P[1] = sin^2(pi/8)  test_runtime.py:53-59
            "coin": "H 0\nM 0\n",                                # fair coin           test_runtime.py:44-50
            "hazard_pair": "X_ERROR(0.1) 0\nX_ERROR(0.3) 1\nM 0 1\n",  # joint chi^2  test_runtime.py:110-121
            "pbinom": "X_ERROR(0.05) 0\nX_ERROR(0.2) 1\nX_ERROR(0.35) 2\nX_ERROR(0.5) 3\nM 0 1 2 3\n",
            "certain": "X_ERROR(1.0) 0\nX_ERROR(0.0) 1\nM 0 1\n",  # p=1 / p=0 sites test_runtime.py:78-107
            "depol1": "DEPOLARIZE1(0.3) 0\nM 0\n",
            "depol2": "DEPOLARIZE2(0.15) 0 1\nM 0 1\n",
            "postselect_half": "H 0\nM 0\nPOSTSELECT rec[-1]\nH 1\nT 1\nH 1\nM 1\n",
        }
        for name, text in laws.items():
            opt = name != "certain"
            prog = compile_circuit(text, optimize=opt)
            np.savez_compressed(ldir / f"{name}.npz",
                                program=np.frombuffer(serialize(prog, name=name).to_npz_bytes(), dtype=np.uint8),
                                circuit=np.array(text))
            print(f"laws/{name}", flush=True)
    if "edges" in which:  # degenerate programs the reference accepts (empty, no records, ...)
        edir = OUT / "edges"
        edir.mkdir(exist_ok=True)
        edges = {
            "empty": "",
            "no_measure": "H 0\nT 0\n",
            "measure_only": "M 0\n",
            "noise_only": "DEPOLARIZE1(0.1) 0\n",
            "empty_detector": "X_ERROR(0.2) 0\nDETECTOR\n",
            "empty_observable": "OBSERVABLE_INCLUDE(0)\n",
            "active_unmeasured": "H 0\nT 0\nH 1\nT 1\nCX 0 1\n",
            "wide_sparse": "H 0\nT 0\nH 0\nM 0\nX_ERROR(0.3) 299\nM 299\nDETECTOR rec[-1]\n",
        }
        for name, text in edges.items():
            prog = compile_circuit(text)
            recs = list(sample(prog, 100, seed=9))
            m = np.array([r.measurements for r in recs], np.uint8).reshape(100, -1)
            d = np.array([r.detectors for r in recs], np.uint8).reshape(100, -1)
            o = np.array([r.observables for r in recs], np.uint8).reshape(100, -1)
            a = np.array([r.accepted for r in recs], np.uint8)
            np.savez_compressed(edir / f"{name}.npz",
                                program=np.frombuffer(serialize(prog, name=name).to_npz_bytes(), dtype=np.uint8),
                                circuit=np.array(text), f_meas=m, f_det=d, f_obs=o, f_acc=a, f_seed=np.array([9]))
            print(f"edges/{name}", flush=True)
    if "probe" in which:  # expectation_probe (runtime.py:951-989) values of the reference
        from framesim.runtime import expectation_probe
        from framesim.pauli import PauliString
        pdir = OUT / "probe"
        pdir.mkdir(exist_ok=True)
        from paper_2604_27058_b200.configs import random_near_clifford
        rng = np.random.default_rng(31)
        circuits = {
            "trivial": "TICK\nZ 0\n",
            "t_state": "H 0\nT 0\n",
            "active_pair": "H 0\nT 0\nH 1\nT 1\nCX 0 1\n",
            "near_clifford": random_near_clifford(7, 4, t_cells=6, seed=5).rsplit("M ", 1)[0],
            "mid_measure": "H 0\nT 0\nH 1\nT 1\nCX 0 1\nH 0\nM 0\nH 2\nT 2\nCX 1 2\n",
        }
        for name, text in circuits.items():
            prog = compile_circuit(text)
            n = prog.n
            labels = [(q, k) for q in range(n) for k in "XYZ"]
            multi = []
            for _ in range(6):
                lab = "".join(rng.choice(list("IXYZ")) for _ in range(n))
                multi.append(lab)
            payload = {"program": np.frombuffer(serialize(prog, name=name).to_npz_bytes(), dtype=np.uint8),
                       "circuit": np.array(text), "final_active": np.array(list(prog.final_active), np.int64)}
            rows = []
            for shot in (0, 1, 2):
                st = ShotState(prog, seed=4)
                run_shot(prog, st, shot=shot)
                obs = [PauliString.single(n, q, k) for q, k in labels] + [PauliString.from_label(l) for l in multi]
                for o in obs:
                    mapped = prog.final_tableau.heisenberg_map(o)
                    word = mapped.hermitian_word()
                    rows.append((shot, np.asarray(word.x, np.uint8), np.asarray(word.z, np.uint8),
                                 int(mapped.hermitian_sign()), float(expectation_probe(prog, st, o))))
            payload["shot"] = np.array([r[0] for r in rows])
            payload["wx"] = np.array([r[1] for r in rows], np.uint8).reshape(len(rows), -1)
            payload["wz"] = np.array([r[2] for r in rows], np.uint8).reshape(len(rows), -1)
            payload["sign"] = np.array([r[3] for r in rows])
            payload["value"] = np.array([r[4] for r in rows])
            np.savez_compressed(pdir / f"{name}.npz", **payload)
            print(f"probe/{name} n={n} k={prog.k_max} probes={len(rows)}", flush=True)
    if "c3deep" in which:  # config 3 (k = 22): 8 trace shots, sketched checkpoints at k >= 20
        text, ps = config_text(3)
        prog = compile_circuit(text, postselect_detectors=ps)
        sched = list(prog.active_schedule)
        big = [i for i, k in enumerate(sched) if k >= 20]
        cps = (big[0], big[len(big) // 2], big[-1])
        t0 = time.time()
        payload = {"program": np.frombuffer(serialize(prog, name="config3_deep").to_npz_bytes(), dtype=np.uint8)}
        payload.update(deep_trace_golden(prog, 8, seed=11, rng=np.random.default_rng(3003), checkpoints=cps))
        np.savez_compressed(OUT / "deep" / "config3_deep.npz", **payload)
        print(f"deep/config3_deep cps={cps} ({time.time() - t0:.1f}s)", flush=True)
    if "c4deep" in which:  # config 4: accepted shots (all 15 post-selections pass), checkpoints at k >= 10
        text, ps = config_text(4)
        prog = compile_circuit(text, postselect_detectors=ps)
        sched = list(prog.active_schedule)
        ks = [i for i, k in enumerate(sched) if k >= 10]
        cps = tuple(sorted({ks[0], ks[len(ks) // 3], ks[2 * len(ks) // 3], ks[-1]}))
        t0 = time.time()
        rng = np.random.default_rng(4004)
        payload = {"program": np.frombuffer(serialize(prog, name="config4_deep").to_npz_bytes(), dtype=np.uint8)}
        payload.update(deep_trace_golden(prog, 8, seed=11, rng=rng, checkpoints=cps,
                                         forced_builder=accepted_forced_builder(prog, text, rng, boost=20.0)))
        np.savez_compressed(OUT / "deep" / "config4_deep.npz", **payload)
        print(f"deep/config4_deep cps={cps} ({time.time() - t0:.1f}s)", flush=True)
    if "renorm" in which:  # renormalize=False (runtime.py:355-366, :389-404, :481)
        rdir = OUT / "renorm"
        rdir.mkdir(exist_ok=True)
        from paper_2604_27058_b200.configs import random_near_clifford
        rng = np.random.default_rng(555)
        cases = {
            "two_fair": ("H 0\nM 0\nH 0\nM 0\n", True),  # |gamma|^2 ||phi||^2 = 0.25 (test_runtime.py:244-249)
            "htm": ("H 0\nT 0\nH 0\nM 0\n", True),
            "unopt_active": ("H 0\nT 0\nH 1\nT 1\nCX 0 1\nH 0\nM 0\nH 1\nM 1\nR_X(0.3) 2\nMX 2\n", False),
            "noise_twice": ("H 0\nT 0\nH 0\nM 0\nDEPOLARIZE1(0.3) 0\nM 0\n", True),
            "near_clifford": (random_near_clifford(7, 6, t_cells=7, seed=21), True),
            "near_clifford_half": (random_near_clifford(8, 5, t_cells=8, seed=22).rsplit("M ", 1)[0]
                                   + "M 0 2 4 6\n", True),
        }
        for i in range(6):
            circ = ftest.random_circuit(rng, int(rng.integers(2, 7)), int(rng.integers(8, 24)), p_noise=0.1,
                                        measure_rate=0.25, max_noncliff=6, reset_rate=0.05)
            cases[f"random{i}"] = (str(circ), bool(i % 3))
        for name, (text, opt) in cases.items():
            t0 = time.time()
            prog = compile_circuit(text, optimize=opt)
            payload = {"program": np.frombuffer(serialize(prog, name=name).to_npz_bytes(), dtype=np.uint8),
                       "circuit": np.array(text)}
            recs = list(sample(prog, 256, seed=8, renormalize=False))
            U, D, O = len(prog.user_records), prog.num_detectors, prog.num_observables
            payload["f_meas"] = np.array([r.measurements for r in recs], np.uint8).reshape(256, U)
            payload["f_det"] = np.array([r.detectors for r in recs], np.uint8).reshape(256, D)
            payload["f_obs"] = np.array([r.observables for r in recs], np.uint8).reshape(256, O)
            payload["f_acc"] = np.array([r.accepted for r in recs], np.uint8)
            payload["f_seed"] = np.array([8])
            # unnormalised states of free shots: gamma, |gamma|^2 ||phi||^2 (= branch probability)
            rows = []
            for shot in range(16):
                st = ShotState(prog, seed=3, renormalize=False)
                run_shot(prog, st, shot=shot)
                rows.append((complex(st.gamma), st.k, st.active_view().copy(), st.records.copy(),
                             st.frame_x.copy(), st.frame_z.copy()))
            ks = {r[1] for r in rows}
            payload["s_gamma"] = np.array([r[0] for r in rows], np.complex128)
            payload["s_total"] = np.array([abs(r[0]) ** 2 * float(np.linalg.norm(r[2]) ** 2) for r in rows])
            payload["s_rec"] = np.array([r[3] for r in rows], np.uint8).reshape(16, -1)
            payload["s_fx"] = np.array([r[4] for r in rows], np.uint8)
            payload["s_fz"] = np.array([r[5] for r in rows], np.uint8)
            payload["s_seed"] = np.array([3])
            if len(ks) == 1:
                payload["s_amps"] = np.array([r[2] for r in rows], np.complex128)
            np.savez_compressed(rdir / f"{name}.npz", **payload)
            print(f"renorm/{name:20s} k_max={prog.k_max} ({time.time() - t0:.1f}s)", flush=True)
    if "accept" in which:  # reference acceptance criterion 3 inputs (test_acceptance.py:131-152)
        from framesim.oracle import dense_run
        from framesim.testing import noise_sites_of, random_fault_plan
        from framesim.circuit import flatten
        t0 = time.time()
        rng = np.random.default_rng(33)
        payload = {}
        for i in range(200):
            n = int(rng.integers(1, 7))
            circ = ftest.random_circuit(rng, n, int(rng.integers(4, 16)), p_noise=0.3, measure_rate=0.25,
                                        max_noncliff=6, reset_rate=0.05, feedforward_rate=0.08)
            plan = random_fault_plan(circ, rng)
            flat = flatten(circ)
            dense = dense_run(flat, fault_plan=plan, seed=9000 + i)
            outcome_plan = {j: int(b) for j, b in enumerate(dense.records)}
            n_sites = len(noise_sites_of(flat))
            modes = np.full(max(n_sites, 0), 2, np.int16)
            for site, case in (plan or {}).items():
                modes[site] = case + 3
            prog = compile_circuit(flat)
            st = ShotState(prog, seed=9000 + i)
            rec = run_shot(prog, st, shot=0, forced_faults=modes if n_sites else None, forced_outcomes=outcome_plan)
            forced = np.full(prog.record_count, -1, np.int8)
            for r, b in outcome_plan.items():
                if r < prog.record_count:
                    forced[r] = b
            key = f"c{i:03d}_"
            payload[key + "program"] = np.frombuffer(serialize(prog, name=f"accept{i:03d}").to_npz_bytes(), dtype=np.uint8)
            payload[key + "modes"] = modes
            payload[key + "forced"] = forced
            payload[key + "seed"] = np.array([9000 + i])
            payload[key + "meas"] = np.asarray(rec.measurements, np.uint8)
            payload[key + "det"] = np.asarray(rec.detectors, np.uint8)
            payload[key + "obs"] = np.asarray(rec.observables, np.uint8)
            payload[key + "oracle_meas"] = np.asarray(dense.user_records, np.uint8)
            payload[key + "rec"] = st.records.copy()
            payload[key + "fx"] = st.frame_x.copy()
            payload[key + "fz"] = st.frame_z.copy()
            payload[key + "gamma"] = np.array([complex(st.gamma)])
            payload[key + "amps"] = st.active_view().copy()
        (OUT / "accept").mkdir(exist_ok=True)
        np.savez_compressed(OUT / "accept" / "criterion3.npz", **payload)
        print(f"accept/criterion3.npz: 200 circuits ({time.time() - t0:.1f}s)", flush=True)
    if "frameref" in which:  # the reference's independent Pauli-frame sampler (oracle.py:407-516)
        from framesim.oracle import pauli_frame_reference_sample
        from framesim.circuit import flatten, parse_circuit
        from paper_2604_27058_b200.configs import rotated_surface_code
        fdir = OUT / "frameref"
        fdir.mkdir(exist_ok=True)
        cases = {
            "config1": (config_text(1)[0], 200_000),                       # config 1 check
            "surface_d5_p5e-3": (rotated_surface_code(5, 5, 5e-3), 200_000),  # boosted rates
            "repetition_d3_r5": (str(ftest.repetition_code_circuit(3, 5, 1e-3)), 1_000_000),  # criterion 4
        }
        for name, (text, shots) in cases.items():
            t0 = time.time()
            circ = flatten(parse_circuit(text))
            prog = compile_circuit(circ)
            det = np.zeros(prog.num_detectors, np.int64)
            obs = np.zeros(prog.num_observables, np.int64)
            chunk = 50_000
            for c0 in range(0, shots, chunk):
                _, d, o = pauli_frame_reference_sample(circ, min(chunk, shots - c0), seed=90404 + c0)
                det += np.asarray(d, np.int64).reshape(-1, prog.num_detectors).sum(0)
                if prog.num_observables:
                    obs += np.asarray(o, np.int64).reshape(-1, prog.num_observables).sum(0)
            np.savez_compressed(fdir / f"{name}.npz",
                                program=np.frombuffer(serialize(prog, name=name).to_npz_bytes(), dtype=np.uint8),
                                det_counts=det, obs_counts=obs, shots=np.array([shots]))
            print(f"frameref/{name}: {shots} frame-sampler shots ({time.time() - t0:.1f}s)", flush=True)
    if "mirrors50" in which:  # acceptance criterion 2 (test_acceptance.py:110-128): 50 exact mirrors
        rng = np.random.default_rng(2024)
        payload = {}
        for i in range(50):
            n = int(rng.integers(1, 9))
            circ = ftest.random_mirror_circuit(rng, n, int(rng.integers(1, 13)))
            prog = compile_circuit(circ)
            payload[f"m{i:02d}"] = np.frombuffer(serialize(prog, name=f"mirror{i:02d}").to_npz_bytes(), dtype=np.uint8)
        (OUT / "accept").mkdir(exist_ok=True)
        np.savez_compressed(OUT / "accept" / "criterion2_mirrors.npz", **payload)
        print("accept/criterion2_mirrors.npz: 50 programs", flush=True)
    if "configs" in which:
        for i in range(5):
            text, ps = config_text(i)
            t0 = time.time()
            prog = compile_circuit(text, postselect_detectors=ps)
            ct = time.time() - t0
            meta = {"config": i, "compile_s": round(ct, 2), "shots": CONFIGS[i]["shots"],
                    "desc": CONFIGS[i]["desc"]}
            P = serialize(prog, name=CONFIGS[i]["name"], meta=meta)
            P.save(PROGS / f"c{i}.npz")
            # reference outputs: bounded by the reference's speed (config 3: ~25 s/shot)
            if i == 3:
                write_case(f"config{i}", prog, "", free_shots=0, trace_shots=1, boost=1.0, meta=meta)
            elif i == 4:
                write_case(f"config{i}", prog, "", free_shots=512, trace_shots=12, boost=20.0, meta=meta,
                           checkpoints=(40, 120))
            else:
                write_case(f"config{i}", prog, "", free_shots=256, trace_shots=12, boost=20.0, meta=meta,
                           checkpoints=(len(prog.instrs) // 3, len(prog.instrs) // 2))


if __name__ == "__main__":
    main(tuple(sys.argv[1:]) or ("toys", "random", "fused", "configs"))
