"""TEST INFRASTRUCTURE ONLY: CPU oracle for the per-shot VM.

``fs_oracle.c`` restates framesim/runtime.py + rng.py (see its header for the
file:line map).  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package; the product (``paper_2604_27058_b200``) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
LIB_PATH = _HERE / "_build" / "libfs_oracle.so"
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> Path:
    """Compile the C restatement (gcc, no FMA contraction, like CPython's arithmetic)."""
    # make does the dependency check (fs_oracle.c and the headers it shares with the engine)
    LIB_PATH.parent.mkdir(exist_ok=True)
    subprocess.check_call(["make", "-s", "-C", str(_HERE)] + (["-B"] if force else []))
    return LIB_PATH


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = C.CDLL(str(LIB_PATH))
            from paper_2604_27058_b200._abi import FsProgDesc, FsSampleOut, FsTraceIn, FsTraceOut

            L.fso_sample.restype = C.c_int
            L.fso_sample.argtypes = [C.POINTER(FsProgDesc), C.c_uint64, C.c_uint64, C.c_uint64,
                                     C.c_uint32, C.POINTER(FsTraceIn), C.POINTER(FsSampleOut),
                                     C.POINTER(FsTraceOut)]
            L.fso_sample_stratum.restype = C.c_int
            L.fso_sample_stratum.argtypes = [C.POINTER(FsProgDesc), C.c_int, C.c_uint64, C.c_uint64, C.c_uint64,
                                             C.c_uint32, C.POINTER(FsSampleOut)]
            L.fso_stratum_weight.restype = C.c_int
            L.fso_stratum_weight.argtypes = [C.POINTER(FsProgDesc), C.c_int, C.POINTER(C.c_double)]
            L.fso_accumulate.restype = C.c_int
            L.fso_accumulate.argtypes = [C.POINTER(FsProgDesc), C.c_uint64, C.c_uint64, C.c_uint64,
                                         C.c_uint32, C.POINTER(C.c_int64)]
            _lib = L
    return _lib


def sample(prog, nshots: int, seed: int = 0, shot0: int = 0, flags: int = 0,
           fault_modes=None, forced=None, stop: int = -1, want_state: bool = False):
    """Run shots [shot0, shot0+nshots) on the CPU oracle.

    Returns (status, HostOutputs, TraceBuffers|None)."""
    from paper_2604_27058_b200._abi import DescHolder, HostOutputs, TraceBuffers

    L = lib()
    h = DescHolder(prog)
    out = HostOutputs(prog, nshots)
    tb = None
    tin = None
    tout = None
    if fault_modes is not None or forced is not None or stop >= 0 or want_state:
        tb = TraceBuffers(prog, nshots, fault_modes, forced, stop, want_state=want_state)
        tin = C.byref(tb.tin)
        tout = C.byref(tb.tout) if tb.tout is not None else None
    st = L.fso_sample(C.byref(h.desc), seed, shot0, nshots, flags, tin, C.byref(out.struct), tout)
    return st, out, tb


def sample_stratum(prog, w: int, nshots: int, seed: int = 0, shot0: int = 0, flags: int = 0):
    """sample(prog, nshots, seed, stratum=StratumSpec(prog, w)) on the CPU oracle: (status, HostOutputs)."""
    from paper_2604_27058_b200._abi import DescHolder, HostOutputs

    L = lib()
    h = DescHolder(prog)
    out = HostOutputs(prog, nshots)
    st = L.fso_sample_stratum(C.byref(h.desc), int(w), seed, shot0, nshots, flags, C.byref(out.struct))
    return st, out


def stratum_weight(prog, w: int) -> float:
    from paper_2604_27058_b200._abi import DescHolder

    h = DescHolder(prog)
    v = C.c_double(0.0)
    if lib().fso_stratum_weight(C.byref(h.desc), int(w), C.byref(v)) != 0:
        raise ValueError(f"stratum fault count {w} exceeds {prog.num_sites} sites")
    return float(v.value)


def accumulate(prog, nshots: int, seed: int = 0, shot0: int = 0, flags: int = 0):
    from paper_2604_27058_b200._abi import DescHolder

    L = lib()
    h = DescHolder(prog)
    n = prog.num_user_records + prog.num_detectors + prog.num_observables + 1
    counts = np.zeros(n, dtype=np.int64)
    st = L.fso_accumulate(C.byref(h.desc), seed, shot0, nshots, flags,
                          counts.ctypes.data_as(C.POINTER(C.c_int64)))
    U, D = prog.num_user_records, prog.num_detectors
    return st, {"shots": nshots, "accepted": int(counts[-1]),
                "measurements": counts[:U], "detectors": counts[U:U + D],
                "observables": counts[U + D:-1]}


def format_records(meas, det, obs, accepted, fmt: str, keep_rejected: bool, weight: float = 1.0,
                   index0: int = 0) -> bytes:
    """CPU restatement of the reference CLI writer (cli.py:66-69, :94-109) over uint8 record arrays
    [shots, ...] -- the checker for the device formatter (fs_format).  The csv header line is not
    included."""
    import numpy as np

    out = []
    idx = index0
    for i in range(len(accepted)):
        if not (accepted[i] or keep_rejected):
            continue
        bits = np.concatenate([meas[i], det[i], obs[i]]).astype(np.uint8)
        if fmt == "bin":
            out.append(np.packbits(bits, bitorder="little").tobytes())
        else:
            text = "".join("1" if b else "0" for b in bits)
            if fmt == "csv":
                out.append(f"{idx},{weight:.17g},{text}\n".encode())
            else:
                if keep_rejected and not accepted[i]:
                    text += " rejected"
                out.append((text + "\n").encode())
        idx += 1
    return b"".join(out)
