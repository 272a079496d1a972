"""Synthetic circuits for the five BASELINE.json configurations.

The reference ships no benchmark circuit files and no surface-code generator
(SURVEY §0 finding 4), so these generators follow the conventions fixed in
SURVEY §8(d).  They emit circuit text in the reference grammar
(``/root/reference/pkg/src/framesim/circuit.py:1-12``); the reference host
compiler turns that text into the bytecode program the GPU engine executes.
``SQRT_X`` is not a reference opcode (``circuit.py:20``) and is emitted as
``H q; S q; H q``, which equals sqrt(X) exactly.

All generators are deterministic functions of their seed (numpy PCG64).
"""
from __future__ import annotations

import numpy as np

_ONEQ = ("H", "S", "S_DAG", "SQRT_X")


def _oneq_line(g: str, q: int) -> list[str]:
    if g == "SQRT_X":
        return [f"H {q}", f"S {q}", f"H {q}"]
    return [f"{g} {q}"]


def _matching(rng: np.random.Generator, qubits) -> list[int]:
    perm = [int(x) for x in rng.permutation(np.asarray(list(qubits)))]
    return perm[: len(perm) // 2 * 2]


def random_near_clifford(n: int, layers: int, t_cells: int | None = None,
                         t_per_layer: int | None = None, seed: int = 0) -> str:
    """Configs 0 and 3: random 1q layer, T gates, CX matching; final M of all qubits."""
    rng = np.random.default_rng(seed)
    cells: set[tuple[int, int]] = set()
    if t_cells is not None:
        flat = rng.choice(layers * n, size=t_cells, replace=False)
        cells = {(int(c) // n, int(c) % n) for c in flat}
    lines: list[str] = []
    for L in range(layers):
        gates = rng.integers(0, len(_ONEQ), size=n)
        for q in range(n):
            lines.extend(_oneq_line(_ONEQ[int(gates[q])], q))
        if t_per_layer is not None:
            for q in sorted(int(x) for x in rng.choice(n, size=t_per_layer, replace=False)):
                lines.append(f"T {q}")
        else:
            for q in range(n):
                if (L, q) in cells:
                    lines.append(f"T {q}")
        m = _matching(rng, range(n))
        if m:
            lines.append("CX " + " ".join(str(q) for q in m))
    lines.append("M " + " ".join(str(q) for q in range(n)))
    return "\n".join(lines) + "\n"


def rotated_surface_code(d: int, rounds: int, p: float, t_qubits=()) -> str:
    """Rotated surface-code Z memory.

    Data (x, y) -> x + d*y.  Plaquette centres (x+1/2, y+1/2), x, y in [-1, d-1];
    X-type if (x+y) even else Z; bulk plaquettes 0 <= x, y <= d-2; boundary
    X-plaquettes only on y in {-1, d-1}, boundary Z-plaquettes only on
    x in {-1, d-1}.  X ancillas visit (nw, ne, sw, se) as CX controls, Z
    ancillas visit (nw, sw, ne, se) as CX targets.  ``t_qubits`` (config 2):
    T on those data qubits before round 1, T_DAG before round 2.
    """
    def data(x, y):
        return x + d * y

    plaqs = []  # (kind, [corner qubits in visiting order or None])
    for y in range(-1, d):
        for x in range(-1, d):
            kind = "X" if (x + y) % 2 == 0 else "Z"
            bulk = 0 <= x <= d - 2 and 0 <= y <= d - 2
            if not bulk:
                if kind == "X" and not (y in (-1, d - 1) and 0 <= x <= d - 2):
                    continue
                if kind == "Z" and not (x in (-1, d - 1) and 0 <= y <= d - 2):
                    continue

            def corner(cx, cy):
                return data(cx, cy) if 0 <= cx < d and 0 <= cy < d else None

            nw, ne = corner(x, y), corner(x + 1, y)
            sw, se = corner(x, y + 1), corner(x + 1, y + 1)
            order = [nw, ne, sw, se] if kind == "X" else [nw, sw, ne, se]
            plaqs.append((kind, order))
    nd = d * d
    anc = [nd + i for i in range(len(plaqs))]
    xanc = [a for a, (k, _) in zip(anc, plaqs) if k == "X"]
    zanc = [a for a, (k, _) in zip(anc, plaqs) if k == "Z"]
    na = len(anc)
    all_anc = " ".join(str(a) for a in anc)
    lines: list[str] = []
    for r in range(rounds):
        if t_qubits and r == 1:
            lines.append("T " + " ".join(str(q) for q in t_qubits))
        if t_qubits and r == 2:
            lines.append("T_DAG " + " ".join(str(q) for q in t_qubits))
        xs = " ".join(str(a) for a in xanc)
        lines.append(f"H {xs}")
        lines.append(f"DEPOLARIZE1({p}) {xs}")
        for step in range(4):
            pairs = []
            for a, (kind, order) in zip(anc, plaqs):
                q = order[step]
                if q is None:
                    continue
                pairs.extend((a, q) if kind == "X" else (q, a))
            tg = " ".join(str(v) for v in pairs)
            lines.append(f"CX {tg}")
            lines.append(f"DEPOLARIZE2({p}) {tg}")
        lines.append(f"H {xs}")
        lines.append(f"DEPOLARIZE1({p}) {xs}")
        lines.append(f"X_ERROR({p}) {all_anc}")
        lines.append(f"M {all_anc}")
        for j, a in enumerate(anc):
            cur = -(na - j)
            if r == 0:
                if a in zanc:
                    lines.append(f"DETECTOR rec[{cur}]")
            else:
                lines.append(f"DETECTOR rec[{cur}] rec[{cur - na}]")
        lines.append(f"X_ERROR({p}) {all_anc}")
        lines.append(f"R {all_anc}")
    lines.append(f"X_ERROR({p}) " + " ".join(str(q) for q in range(nd)))
    lines.append("M " + " ".join(str(q) for q in range(nd)))
    for j, (a, (kind, order)) in enumerate(zip(anc, plaqs)):
        if kind != "Z":
            continue
        refs = [f"rec[{q - nd}]" for q in order if q is not None]
        refs.append(f"rec[{-(nd + na - j)}]")
        lines.append("DETECTOR " + " ".join(refs))
    obs = [f"rec[{data(x, 0) - nd}]" for x in range(d)]
    lines.append("OBSERVABLE_INCLUDE(0) " + " ".join(obs))
    return "\n".join(lines) + "\n"


def cultivation_like(n: int = 50, layers: int = 60, p: float = 5e-4, register: int = 12,
                     seed: int = 0) -> str:
    """Config 4, magic-register variant (SURVEY §0 finding 1, §8(d)).

    Every layer: random 1q Clifford + DEPOLARIZE1 on every qubit; layers with
    L % 3 == 0 get T or T_DAG (fair coin) on 2 distinct qubits of the
    ``register`` (qubits 0..register-1); CX matchings are drawn separately
    inside the register and inside the rest, followed by DEPOLARIZE2; every
    4th layer (L % 4 == 3) measures 4 random qubits, adds a parity detector and
    resets them.  Final Z measurement of all qubits.  ``register=n`` gives the
    literal construction (k_max = 35, infeasible).
    """
    rng = np.random.default_rng(seed)
    lines: list[str] = []
    allq = " ".join(str(q) for q in range(n))
    for L in range(layers):
        gates = rng.integers(0, len(_ONEQ), size=n)
        for q in range(n):
            lines.extend(_oneq_line(_ONEQ[int(gates[q])], q))
        lines.append(f"DEPOLARIZE1({p}) {allq}")
        if L % 3 == 0:
            qs = rng.choice(register, size=2, replace=False)
            for q in qs:
                g = "T" if rng.random() < 0.5 else "T_DAG"
                lines.append(f"{g} {int(q)}")
        if register < n:
            m = _matching(rng, range(register)) + _matching(rng, range(register, n))
        else:
            m = _matching(rng, range(n))
        tg = " ".join(str(q) for q in m)
        lines.append(f"CX {tg}")
        lines.append(f"DEPOLARIZE2({p}) {tg}")
        if L % 4 == 3:
            qs = " ".join(str(int(q)) for q in rng.choice(n, size=4, replace=False))
            lines.append(f"M {qs}")
            lines.append("DETECTOR rec[-1] rec[-2] rec[-3] rec[-4]")
            lines.append(f"R {qs}")
    lines.append(f"M {allq}")
    return "\n".join(lines) + "\n"


CONFIGS = {
    0: dict(name="c0_random16_6T", shots=100_000,
            desc="n=16, 30 random layers, 6 T, noiseless, final M (k_max<=6)"),
    1: dict(name="c1_surface_d5_r5", shots=10_000_000,
            desc="rotated surface code d=5 r=5 p=1e-3 Z-memory (k=0, frame-only)"),
    2: dict(name="c2_surface_d3_r3_T", shots=10_000_000,
            desc="rotated surface code d=3 r=3 p=1e-3 + 4 T / 4 T_DAG between rounds (k_max=4)"),
    3: dict(name="c3_random22_320T", shots=1_000,
            desc="n=22, 40 layers x 8 T, noiseless, final M (k=22, HBM-resident)"),
    4: dict(name="c4_cultivation_m12", shots=100_000_000,
            desc="n=50, 60 layers, ~40 T/T_DAG in a 12-qubit register, p=5e-4, "
                 "15 post-selected parity detectors (k_max=12)"),
}


def config_text(i: int, seed: int = 0) -> tuple[str, tuple]:
    """(circuit text, postselect_detectors) for BASELINE.json config ``i``."""
    if i == 0:
        return random_near_clifford(16, 30, t_cells=6, seed=seed), ()
    if i == 1:
        return rotated_surface_code(5, 5, 1e-3), ()
    if i == 2:
        rng = np.random.default_rng(seed + 2000)
        tq = sorted(int(q) for q in rng.choice(9, size=4, replace=False))
        return rotated_surface_code(3, 3, 1e-3, t_qubits=tq), ()
    if i == 3:
        return random_near_clifford(22, 40, t_per_layer=8, seed=seed), ()
    if i == 4:
        return cultivation_like(seed=seed), tuple(range(15))
    raise KeyError(i)
