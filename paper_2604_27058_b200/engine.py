"""Python handle over the C-ABI: one compiled program resident on the GPU.

``DeviceProgram`` is the host-side object behind the reference-shaped API in
``runtime.py``; it owns an ``fs_prog*`` (``include/fs_sampler.h``).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _abi
from ._abi import DescHolder, FsSampleOut, HostOutputs, TraceBuffers, vptr
from ._lib import EngineUnavailable, last_error, lib
from .program import Program, as_program


class ShotError(RuntimeError):
    """Mirror of ``framesim.runtime.ShotError`` (runtime.py:51-52)."""


def raise_for_status(status: int) -> None:
    if status == _abi.FS_OK:
        return
    if status == _abi.FS_ERR_SHOT_NAN:
        raise ShotError("NaN amplitude encountered at an active measurement")
    if status == _abi.FS_ERR_SHOT_FORCED:
        raise ShotError("forced outcome has probability below BRANCH_FLOOR (probability 0)")
    if status == _abi.FS_ERR_ARG:
        raise ValueError(last_error())
    raise EngineUnavailable(f"CUDA engine error {status}: {last_error()}")


class DeviceProgram:
    """A serialized program uploaded to the current CUDA device."""

    def __init__(self, prog):
        self.prog: Program = as_program(prog)
        self._lib = lib()
        self._desc = DescHolder(self.prog)
        h = C.c_void_p()
        rc = self._lib.fs_program_create(C.byref(self._desc.desc), C.byref(h))
        if rc != _abi.FS_OK:
            raise EngineUnavailable(f"fs_program_create failed ({rc}): {last_error()}")
        self._h = h

    def close(self) -> None:
        if getattr(self, "_h", None):
            self._lib.fs_program_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover - best effort
        try:
            self.close()
        except Exception:
            pass

    def jit_status(self) -> str:
        """State of the program-specialised frame kernel ("ready ...", "not built", "failed: ...")."""
        f = self._lib.fs_debug_jit_status
        f.restype = C.c_char_p
        f.argtypes = [C.c_void_p]
        return f(self._h).decode()

    def segment_counts(self) -> list[int]:
        """Diagnostics of the last segmented call: shots entering each post-select segment."""
        buf = (C.c_uint32 * 4096)()
        f = self._lib.fs_debug_seg_counts
        f.argtypes = [C.c_void_p, C.POINTER(C.c_uint32), C.c_int]
        n = f(self._h, buf, 4096)
        return [int(buf[i]) for i in range(min(max(n, 0), 4096))]

    def engine(self, flags: int = 0) -> str:
        return {0: "general", 1: "frame", 2: "hbm"}[self._lib.fs_program_engine(self._h, flags)]

    # -- host buffers (C-ABI does H2D/D2H) ----------------------------------------------
    def sample_host(self, nshots: int, seed: int = 0, shot0: int = 0, flags: int = 0,
                    fault_modes=None, forced=None, stop: int = -1, want_state: bool = False,
                    check: bool = True, checkpoints=None):
        """Returns (status, HostOutputs, TraceBuffers|None).  ``checkpoints``: instruction counts
        at which the state is also recorded (TraceBuffers.checkpoint(j))."""
        if nshots < 1:
            raise ValueError("shots must be >= 1")
        out = HostOutputs(self.prog, nshots)
        status = np.zeros(1, dtype=np.int32)
        out.struct.status = status.ctypes.data_as(C.POINTER(C.c_int32))
        tb = None
        tin = tout = None
        if fault_modes is not None or forced is not None or stop >= 0 or want_state or checkpoints is not None:
            tb = TraceBuffers(self.prog, nshots, fault_modes, forced, stop, want_state=want_state,
                              checkpoints=checkpoints)
            tin = C.byref(tb.tin)
            tout = C.byref(tb.tout) if tb.tout is not None else None
        rc = self._lib.fs_sample_host(self._h, seed, shot0, nshots, flags, tin, C.byref(out.struct), tout)
        if rc < 0 or (check and rc != 0):
            raise_for_status(rc)
        return rc, out, tb

    # -- device buffers (torch tensors; the benchmark / streaming path) -------------------
    def alloc_device_outputs(self, nshots: int, device=None):
        import torch

        W = (nshots + 31) // 32
        p = self.prog
        dev = device or torch.device("cuda")
        t = {
            "meas": torch.empty((max(p.num_user_records, 1), W), dtype=torch.int32, device=dev),
            "det": torch.empty((max(p.num_detectors, 1), W), dtype=torch.int32, device=dev),
            "obs": torch.empty((max(p.num_observables, 1), W), dtype=torch.int32, device=dev),
            "accepted": torch.empty(W, dtype=torch.int32, device=dev),
            "error": torch.empty(W, dtype=torch.int32, device=dev),
            "status": torch.zeros(1, dtype=torch.int32, device=dev),
        }
        return t

    def sample_device(self, nshots: int, out: dict, seed: int = 0, shot0: int = 0, flags: int = 0,
                      stream=None) -> None:
        """Asynchronous launch into preallocated device tensors (see alloc_device_outputs)."""
        import torch

        o = FsSampleOut()
        o.meas = vptr(out["meas"].data_ptr(), C.c_uint32)
        o.det = vptr(out["det"].data_ptr(), C.c_uint32)
        o.obs = vptr(out["obs"].data_ptr(), C.c_uint32)
        o.accepted = vptr(out["accepted"].data_ptr(), C.c_uint32)
        o.error = vptr(out["error"].data_ptr(), C.c_uint32)
        o.status = vptr(out["status"].data_ptr(), C.c_int32)
        s = stream if stream is not None else torch.cuda.current_stream()
        rc = self._lib.fs_sample(self._h, seed, shot0, nshots, flags, None, C.byref(o), None,
                                 C.c_void_p(s.cuda_stream))
        if rc != 0:
            raise_for_status(rc)

    def format_device(self, nshots: int, out: dict, fmt: int, keep_rejected: bool, index0: int,
                      weight_text: str, dst, stream=None) -> tuple[int, int]:
        """fs_format: reference CLI bytes of the shots in `out` into the uint8 device tensor `dst`.
        Returns (bytes, records) written; synchronizes `stream`."""
        import torch

        o = FsSampleOut()
        o.meas = vptr(out["meas"].data_ptr(), C.c_uint32)
        o.det = vptr(out["det"].data_ptr(), C.c_uint32)
        o.obs = vptr(out["obs"].data_ptr(), C.c_uint32)
        o.accepted = vptr(out["accepted"].data_ptr(), C.c_uint32)
        s = stream if stream is not None else torch.cuda.current_stream()
        nb, nk = C.c_uint64(0), C.c_uint64(0)
        rc = self._lib.fs_format(self._h, C.byref(o), nshots, fmt, 1 if keep_rejected else 0, index0,
                                 weight_text.encode(), C.c_void_p(dst.data_ptr()), dst.numel(), C.byref(nb),
                                 C.byref(nk), C.c_void_p(s.cuda_stream))
        if rc != 0:
            raise_for_status(rc)
        return int(nb.value), int(nk.value)

    def format_bound(self, nshots: int, fmt: int, index0: int, weight_text: str) -> int:
        return int(self._lib.fs_format_bound(self._h, nshots, fmt, index0, weight_text.encode()))

    def accumulate_device(self, nshots: int, counts, seed: int = 0, shot0: int = 0, flags: int = 0,
                          stream=None) -> None:
        import torch

        s = stream if stream is not None else torch.cuda.current_stream()
        rc = self._lib.fs_accumulate(self._h, seed, shot0, nshots, flags,
                                     C.c_void_p(counts.data_ptr()), C.c_void_p(s.cuda_stream))
        if rc != 0:
            raise_for_status(rc)

    def accumulate(self, nshots: int, seed: int = 0, shot0: int = 0, flags: int = 0) -> dict:
        import torch

        p = self.prog
        nrows = p.num_user_records + p.num_detectors + p.num_observables
        counts = torch.zeros(nrows + 1, dtype=torch.int64, device="cuda")
        self.accumulate_device(nshots, counts, seed, shot0, flags)
        c = counts.cpu().numpy()
        U, D = p.num_user_records, p.num_detectors
        return {"shots": nshots, "accepted": int(c[-1]),
                "measurements": c[:U], "detectors": c[U:U + D], "observables": c[U + D:-1]}

    # -- stratified importance sampling (runtime.py:886-945) ------------------------------
    def stratum_weight(self, w: int) -> float:
        """StratumSpec(prog, w).weight = Pr[W = w] (ValueError when w exceeds the site count)."""
        v = C.c_double(0.0)
        rc = self._lib.fs_stratum_weight(self._h, int(w), C.byref(v))
        if rc != 0:
            raise ValueError(self._lib.fs_last_error().decode())
        return float(v.value)

    def sample_stratum_host(self, w: int, nshots: int, seed: int = 0, shot0: int = 0, flags: int = 0,
                            check: bool = True):
        """Shots conditioned on exactly w faults: (status, HostOutputs)."""
        if nshots < 1:
            raise ValueError("shots must be >= 1")
        out = HostOutputs(self.prog, nshots)
        status = np.zeros(1, dtype=np.int32)
        out.struct.status = status.ctypes.data_as(C.POINTER(C.c_int32))
        rc = self._lib.fs_sample_stratum_host(self._h, int(w), seed, shot0, nshots, flags, C.byref(out.struct))
        if rc < 0:
            raise ValueError(self._lib.fs_last_error().decode())
        if check and rc != 0:
            raise_for_status(rc)
        return rc, out

    def sample_stratum_device(self, w: int, nshots: int, out: dict, seed: int = 0, shot0: int = 0,
                              flags: int = 0, stream=None) -> None:
        import torch

        o = FsSampleOut()
        o.meas = vptr(out["meas"].data_ptr(), C.c_uint32)
        o.det = vptr(out["det"].data_ptr(), C.c_uint32)
        o.obs = vptr(out["obs"].data_ptr(), C.c_uint32)
        o.accepted = vptr(out["accepted"].data_ptr(), C.c_uint32)
        o.error = vptr(out["error"].data_ptr(), C.c_uint32)
        o.status = vptr(out["status"].data_ptr(), C.c_int32)
        s = stream if stream is not None else torch.cuda.current_stream()
        rc = self._lib.fs_sample_stratum(self._h, int(w), seed, shot0, nshots, flags, C.byref(o),
                                         C.c_void_p(s.cuda_stream))
        if rc < 0:
            raise ValueError(self._lib.fs_last_error().decode())
        if rc != 0:
            raise_for_status(rc)

    def accumulate_stratum(self, w: int, nshots: int, seed: int = 0, shot0: int = 0, flags: int = 0) -> dict:
        import torch

        p = self.prog
        nrows = p.num_user_records + p.num_detectors + p.num_observables
        counts = torch.zeros(nrows + 1, dtype=torch.int64, device="cuda")
        s = torch.cuda.current_stream()
        rc = self._lib.fs_accumulate_stratum(self._h, int(w), seed, shot0, nshots, flags,
                                             C.c_void_p(counts.data_ptr()), C.c_void_p(s.cuda_stream))
        if rc < 0:
            raise ValueError(self._lib.fs_last_error().decode())
        if rc != 0:
            raise_for_status(rc)
        c = counts.cpu().numpy()
        U, D = p.num_user_records, p.num_detectors
        return {"shots": nshots, "accepted": int(c[-1]),
                "measurements": c[:U], "detectors": c[U:U + D], "observables": c[U + D:-1]}
