"""Hand-built bytecode programs (no reference compiler needed) for engine-vs-oracle tests.

The instruction classes carry the names and fields ``program.serialize`` reads from the reference's
dataclasses (backend.py:107-241); a program is a list of them plus the BytecodeProgram attributes
(backend.py:254-269).  Used for the block engine's star groups: runs of ArrayGates through one
pivot axis, with FrameGates in between and an optional closing ArrayRot, in every shape the host
grouping (fs_sampler.cu fs_program_create) accepts or has to refuse.
"""
from __future__ import annotations

import math
from types import SimpleNamespace

import numpy as np

from paper_2604_27058_b200.program import serialize


def _ins(_cls, **kw):
    return type(_cls, (), kw)()


def star_program(k: int, seed: int, ngroups: int = 6, dormant: int = 3):
    """Expand to k active axes, `ngroups` random gate runs (star-shaped and not), then measure every
    axis.  A PostSelect on a record that is always 0 routes the program through the segmented
    engine; random coins on every qubit make the frame (ArrayRot / Expand parities) shot-dependent."""
    rng = np.random.default_rng(seed)
    n = k + dormant
    ins, sched = [], []
    kk = 0
    rec = 0

    def emit(x):
        ins.append(x)
        sched.append(kk)

    def frame_gates(m):
        gs = []
        for _ in range(m):
            g = ["H", "S", "S_DAG", "CX", "CZ", "SWAP", "X"][rng.integers(0, 7)]
            a = int(rng.integers(0, n))
            b = None
            if g in ("CX", "CZ", "SWAP"):
                b = int((a + 1 + rng.integers(0, n - 1)) % n)
            gs.append((g, a, b))
        emit(_ins("FrameGates", gates=gs))

    emit(_ins("MeasDormantStatic", virt=n - 1, record=rec, flip=0)); rec += 1
    emit(_ins("PostSelectIns", kind="record", ref=0, required=0))
    for q in range(n):
        emit(_ins("MeasDormantRandom", virt=q, record=rec, flip=int(rng.integers(0, 2)))); rec += 1
    frame_gates(2 * n)
    for j in range(k):
        kk = j + 1
        emit(_ins("Expand", virt=j, axis=j, size=1 << j, fused=True, angle=float(rng.uniform(0, 2 * math.pi))))
        if rng.random() < 0.5:
            frame_gates(3)
    size = 1 << k
    cuts = []  # instruction counts right after a run closed by H or ArrayRot (no group spans them)

    def gate(g, a, b=None):
        emit(_ins("ArrayGate", gate=g, va=a, vb=b, axa=a, axb=b, size=size))

    for _ in range(ngroups):
        a = int(rng.integers(0, k))
        others = [x for x in range(k) if x != a]
        shape = int(rng.integers(0, 5))
        if shape == 4 and k >= 3:  # not a star: controls differ, targets repeat
            for _ in range(4):
                c, t = rng.choice(k, 2, replace=False)
                gate("CX" if rng.random() < 0.5 else "CZ", int(c), int(t))
            continue
        for _ in range(int(rng.integers(1, 2 * k + 2))):
            r = rng.random()
            o = int(rng.choice(others)) if others else None
            if o is None or r < 0.15:
                gate("S" if rng.random() < 0.5 else "S_DAG", a)
            elif r < 0.55:
                gate("CX", a, o)
            elif r < 0.8:
                gate("CZ", a, o)
            else:
                gate("CZ", o, a)
            if rng.random() < 0.3:
                frame_gates(int(rng.integers(1, 4)))
        if shape in (0, 1):
            gate("H", a)
        if shape in (0, 2):
            if rng.random() < 0.5:
                frame_gates(2)
            emit(_ins("ArrayRot", virt=int(rng.integers(0, n)), axis=int(rng.integers(0, k)) if shape == 2 else a,
                      angle=float(rng.uniform(0, 2 * math.pi)), size=size))
        if shape in (0, 1, 2):
            cuts.append(len(ins))
        if rng.random() < 0.4:
            frame_gates(4)
    s2 = 1.0 / math.sqrt(2.0)
    for axis in range(k - 1, -1, -1):
        u = ((1.0, 0.0), (0.0, 1.0)) if rng.random() < 0.5 else ((s2, s2), (s2, -s2))
        kk = axis
        emit(_ins("MeasCollapse", virt=axis, axis=axis, record=rec, flip=0, size=2 << axis, u=u, pre_gates=[])); rec += 1
    prog = SimpleNamespace(n=n, k_max=k, record_count=rec, num_detectors=0, num_observables=0, instrs=ins,
                           sites=[], cum_hazard=[0.0], user_records=list(range(rec)), active_schedule=sched)
    return serialize(prog, name=f"star_k{k}_s{seed}", meta={"cuts": sorted(set(cuts))})
