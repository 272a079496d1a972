"""expectation_probe (runtime.py:951-989) against the reference's values.

Goldens (tests/golden/probe, make_golden.py "probe"): per circuit, shot and observable the
reference's Heisenberg-mapped Hermitian word (x, z), sign and ``expectation_probe`` value after
``run_shot(prog, ShotState(prog, seed=4), shot)``.  Here the state is rebuilt by our run_shot
(reference stream) and the traversal runs on the GPU (fs_probe).
"""
from __future__ import annotations

import io
from pathlib import Path

import numpy as np
import pytest

from paper_2604_27058_b200.program import Program

PDIR = Path(__file__).parent / "golden" / "probe"
CASES = sorted(p.stem for p in PDIR.glob("*.npz"))


def _load(name):
    with np.load(PDIR / f"{name}.npz", allow_pickle=False) as z:
        g = {k: z[k] for k in z.files}
    g["prog"] = Program.load(io.BytesIO(g["program"].tobytes()))
    return g


def test_probe_needs_reference_program():
    from paper_2604_27058_b200 import runtime

    g = _load(CASES[0])
    with pytest.raises(TypeError):
        runtime.expectation_probe(g["prog"], None, None)


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_gpu_probe_matches_reference(cuda, name):
    from paper_2604_27058_b200 import runtime

    g = _load(name)
    P = g["prog"]
    states = {}
    for shot in sorted(set(g["shot"].tolist())):
        st = runtime.ShotState(P, seed=4)
        runtime.run_shot(P, st, shot=int(shot), seed=4)
        states[int(shot)] = st
    for i in range(len(g["value"])):
        st = states[int(g["shot"][i])]
        v = runtime.probe_mapped(st, g["wx"][i], g["wz"][i], int(g["sign"][i]), g["final_active"])
        assert abs(v - float(g["value"][i])) < 1e-10, (i, v, float(g["value"][i]))
