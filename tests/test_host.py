"""CPU-only tests: serialized program format, C-ABI library surface, host-side logic."""
from __future__ import annotations

import ctypes as C
import io
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

from goldens import case_names, load
from paper_2604_27058_b200 import _abi
from paper_2604_27058_b200.configs import CONFIGS, config_text
from paper_2604_27058_b200.program import Program

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "fs_sampler.h"


def test_program_npz_round_trip():
    for name in case_names()[:10]:
        P = load(name)["prog"]
        Q = Program.load(io.BytesIO(P.to_npz_bytes()))
        for k in Program._ARRAYS:
            np.testing.assert_array_equal(getattr(P, k), getattr(Q, k))
        for k in Program._SCALARS:
            assert getattr(P, k) == getattr(Q, k)


def test_config_programs_shapes():
    """Shapes of the five BASELINE configs as compiled by the reference compiler."""
    progs = {i: Program.load(ROOT / "paper_2604_27058_b200" / "programs" / f"c{i}.npz") for i in range(5)}
    assert progs[0].n == 16 and progs[0].k_max == 6
    assert progs[1].n == 49 and progs[1].k_max == 0 and progs[1].num_detectors == 120
    assert progs[1].num_sites == 785 and progs[1].num_instrs == 584
    assert progs[2].n == 17 and progs[2].k_max == 4 and progs[2].num_detectors == 24
    assert progs[3].n == 22 and progs[3].k_max == 22 and progs[3].num_sites == 0
    assert progs[4].n == 50 and progs[4].k_max == 12 and progs[4].num_detectors == 15
    assert progs[4].has_postselect and progs[4].num_sites == 4500
    for i in range(5):
        assert progs[i].meta["config"] == i


def test_config_generators_deterministic():
    for i in range(5):
        a, pa = config_text(i)
        b, pb = config_text(i)
        assert a == b and pa == pb
    assert CONFIGS[1]["shots"] == 10_000_000


def test_slot_allocation_is_valid():
    """Every bit read after being written has a slot, and no two live bits share one."""
    for name in case_names():
        P = load(name)["prog"]
        R = P.record_count
        ops = P.instrs[:, 0] & 0xFF
        live = {}
        for i in range(P.num_instrs):
            w = P.instrs[i]
            op = int(ops[i])
            reads = []
            if op == 10:
                reads = [int(w[3])]
            elif op in (12, 13):
                reads = [int(x) for x in P.reclists[w[2]:w[2] + w[3]]]
            elif op == 14:
                reads = [R + int(w[2]) if w[1] == 0 else int(w[2])]
            for b in reads:
                s = P.bit_slot[b]
                assert s >= 0, (name, b)
                assert live.get(s) == b, (name, i, b, live.get(s))
            writes = []
            if op in (5, 6, 7, 8):
                writes = [int(w[3])]
            elif op == 12:
                writes = [R + int(w[1])]
            for b in writes:
                if P.bit_slot[b] >= 0:
                    live[int(P.bit_slot[b])] = b


def _header_functions():
    txt = HEADER.read_text()
    return re.findall(r"^\s*(?:int|void|const char\*)\s+(fs_\w+)\s*\(", txt, re.M)


def test_engine_library_exports_abi():
    """The in-tree C-ABI library loads (no GPU needed) and exports every header symbol."""
    from paper_2604_27058_b200 import _lib

    L = _lib.lib()
    names = _header_functions()
    assert {"fs_program_create", "fs_sample", "fs_sample_host", "fs_accumulate",
            "fs_program_destroy", "fs_last_error", "fs_abi_version", "fs_program_engine"} <= set(names)
    for nm in names:
        assert hasattr(L, nm), nm
    assert L.fs_abi_version() == _abi.FS_ABI_VERSION


def test_abi_struct_layout_matches_header(tmp_path):
    """ctypes mirrors (paper_2604_27058_b200/_abi.py) == C layout of include/fs_sampler.h."""
    src = tmp_path / "lay.c"
    structs = {"fs_prog_desc": _abi.FsProgDesc, "fs_trace_in": _abi.FsTraceIn,
               "fs_trace_out": _abi.FsTraceOut, "fs_sample_out": _abi.FsSampleOut}
    lines = ['#include <stdio.h>', '#include <stddef.h>', f'#include "{HEADER}"', "int main(void){"]
    for cname, py in structs.items():
        lines.append(f'printf("{cname} %zu\\n", sizeof({cname}));')
        for fname, _ in py._fields_:
            lines.append(f'printf("{cname}.{fname} %zu\\n", offsetof({cname}, {fname}));')
    lines.append("return 0;}")
    src.write_text("\n".join(lines))
    exe = tmp_path / "lay"
    subprocess.check_call(["gcc", "-o", str(exe), str(src)])
    got = dict(ln.split() for ln in subprocess.check_output([str(exe)], text=True).splitlines())
    for cname, py in structs.items():
        assert int(got[cname]) == C.sizeof(py), cname
        for fname, _ in py._fields_:
            assert int(got[f"{cname}.{fname}"]) == getattr(py, fname).offset, (cname, fname)


def test_header_flags_match_python():
    txt = HEADER.read_text()
    for nm in ("FS_RNG_SPLITMIX", "FS_NO_RENORM", "FS_FORCE_GENERAL", "FS_FORCE_HBM"):
        m = re.search(rf"#define {nm}\s+(\d+)u", txt)
        assert m and int(m.group(1)) == getattr(_abi, nm), nm


def test_engine_fails_loudly_without_gpu():
    """No CPU fallback: creating a device program without CUDA raises, never silently succeeds."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2604_27058_b200.engine import DeviceProgram, EngineUnavailable

    with pytest.raises(EngineUnavailable):
        DeviceProgram(load("toy_htm")["prog"])


def test_unpack_layout():
    words = np.array([[0b1011, 1 << 31]], dtype=np.uint32)
    bits = _abi.HostOutputs.unpack(words, 64)
    assert bits.shape == (64, 1)
    assert bits[:4, 0].tolist() == [1, 1, 0, 1] and bits[63, 0] == 1 and bits[4:63, 0].sum() == 0


@pytest.mark.parametrize("name", ["config1", "aff_mixed", "aff_rep_psel", "toy_certain", "mirror00", "rand06", "aff_surface_d7"])
def test_affine_kernel_source_compiles(name, tmp_path):
    """The affine frame kernel generated for a frame-only program (fs_affine.cuh) compiles for
    sm_100a without a GPU (nvcc -cubin): the GPU tests then only exercise its behaviour."""
    from paper_2604_27058_b200 import _lib
    from paper_2604_27058_b200._abi import DescHolder

    P = load(name)["prog"]
    h = DescHolder(P)
    L = _lib.lib()
    L.fs_debug_aff_source.argtypes = [C.c_void_p, C.c_char_p, C.c_size_t]
    n = L.fs_debug_aff_source(C.byref(h.desc), None, 0)
    assert n > 0, n
    buf = C.create_string_buffer(n + 1)
    L.fs_debug_aff_source(C.byref(h.desc), buf, n + 1)
    src = tmp_path / f"aff_{name}.cu"
    src.write_text(buf.value.decode())
    inc = ROOT / "paper_2604_27058_b200" / "csrc"
    r = subprocess.run(["nvcc", "-cubin", "-arch=sm_100a", "-std=c++17", "-I", str(inc), "-I", str(ROOT / "include"),
                        "-o", str(tmp_path / "k.cubin"), str(src)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-2000:]
    sass = subprocess.run(["cuobjdump", "-sass", str(tmp_path / "k.cubin")], capture_output=True, text=True).stdout
    assert "fs_aff_frame" in sass
