"""ctypes mirror of ``include/fs_sampler.h`` (structs, flags, status codes).

Host-side plumbing only: it builds the plain-pointer descriptors the C ABI
takes.  Every array referenced by a descriptor is kept alive by the returned
holder object.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

FS_ABI_VERSION = 2
FS_RNG_PHILOX = 0
FS_RNG_SPLITMIX = 1
FS_NO_RENORM = 2
FS_FORCE_GENERAL = 4
FS_FORCE_HBM = 8
FS_NO_JIT = 16
FS_FORCE_SEGMENTED = 32

FS_OK = 0
FS_ERR_ARG = -1
FS_ERR_CUDA = -2
FS_ERR_SHOT_NAN = 1
FS_ERR_SHOT_FORCED = 2

_i32p = C.POINTER(C.c_int32)
_u32p = C.POINTER(C.c_uint32)
_f64p = C.POINTER(C.c_double)


class FsProgDesc(C.Structure):
    _fields_ = [
        ("abi_version", C.c_int32), ("n", C.c_int32), ("k_max", C.c_int32),
        ("num_instrs", C.c_int32), ("record_count", C.c_int32),
        ("num_user_records", C.c_int32), ("num_detectors", C.c_int32),
        ("num_observables", C.c_int32), ("num_sites", C.c_int32), ("num_slots", C.c_int32),
        ("num_fparams", C.c_int32), ("num_gates", C.c_int32), ("num_paulis", C.c_int32),
        ("num_reclists", C.c_int32), ("num_cases", C.c_int32), ("num_plans", C.c_int32),
        ("instrs", _i32p), ("schedule", _i32p), ("fparams", _f64p), ("gates", _u32p),
        ("paulis", _u32p), ("reclists", _i32p), ("site_prob", _f64p),
        ("site_case_off", _i32p), ("case_cum", _f64p), ("case_pauli_off", _i32p),
        ("cum_hazard", _f64p), ("plans", _i32p), ("user_records", _i32p),
        ("record_out", _i32p), ("bit_slot", _i32p),
    ]


class FsTraceIn(C.Structure):
    _fields_ = [("fault_modes", C.POINTER(C.c_int16)), ("forced", C.POINTER(C.c_int8)),
                ("stop", C.c_int32), ("ncheckpoints", C.c_int32), ("checkpoints", C.POINTER(C.c_int32))]


class FsTraceOut(C.Structure):
    _fields_ = [("frame_x", C.POINTER(C.c_uint8)), ("frame_z", C.POINTER(C.c_uint8)),
                ("gamma", _f64p), ("amps", _f64p), ("draws", _u32p), ("records", C.POINTER(C.c_uint8)),
                ("cp_valid", C.POINTER(C.c_uint8)), ("cp_frame_x", C.POINTER(C.c_uint8)),
                ("cp_frame_z", C.POINTER(C.c_uint8)), ("cp_gamma", _f64p), ("cp_amps", _f64p)]


class FsSampleOut(C.Structure):
    _fields_ = [("meas", _u32p), ("det", _u32p), ("obs", _u32p), ("accepted", _u32p),
                ("error", _u32p), ("status", _i32p)]


def _ptr(arr: np.ndarray | None, ctype):
    if arr is None:
        return C.cast(None, C.POINTER(ctype))
    assert arr.flags["C_CONTIGUOUS"]
    return arr.ctypes.data_as(C.POINTER(ctype))


def vptr(addr: int | None, ctype):
    """Pointer from a raw (e.g. device) address."""
    return C.cast(C.c_void_p(addr or None), C.POINTER(ctype))


class DescHolder:
    """Keeps the numpy arrays a descriptor points into alive."""

    def __init__(self, prog):
        self.arrays = {}

        def keep(name, arr, dtype):
            a = np.ascontiguousarray(arr, dtype=dtype)
            if a.size == 0:
                a = np.zeros(1, dtype=dtype)  # never hand out NULL for an empty table
            self.arrays[name] = a
            return a

        d = FsProgDesc()
        d.abi_version = FS_ABI_VERSION
        d.n = prog.n
        d.k_max = prog.k_max
        d.num_instrs = prog.num_instrs
        d.record_count = prog.record_count
        d.num_user_records = prog.num_user_records
        d.num_detectors = prog.num_detectors
        d.num_observables = prog.num_observables
        d.num_sites = prog.num_sites
        d.num_slots = prog.num_slots
        d.num_fparams = int(prog.fparams.size)
        d.num_gates = int(prog.gates.size)
        d.num_paulis = int(prog.paulis.size)
        d.num_reclists = int(prog.reclists.size)
        d.num_cases = int(prog.case_cum.size)
        d.num_plans = int(prog.plans.shape[0])
        d.instrs = _ptr(keep("instrs", prog.instrs, np.int32), C.c_int32)
        d.schedule = _ptr(keep("schedule", prog.schedule, np.int32), C.c_int32)
        d.fparams = _ptr(keep("fparams", prog.fparams, np.float64), C.c_double)
        d.gates = _ptr(keep("gates", prog.gates, np.uint32), C.c_uint32)
        d.paulis = _ptr(keep("paulis", prog.paulis, np.uint32), C.c_uint32)
        d.reclists = _ptr(keep("reclists", prog.reclists, np.int32), C.c_int32)
        d.site_prob = _ptr(keep("site_prob", prog.site_prob, np.float64), C.c_double)
        d.site_case_off = _ptr(keep("site_case_off", prog.site_case_off, np.int32), C.c_int32)
        d.case_cum = _ptr(keep("case_cum", prog.case_cum, np.float64), C.c_double)
        d.case_pauli_off = _ptr(keep("case_pauli_off", prog.case_pauli_off, np.int32), C.c_int32)
        d.cum_hazard = _ptr(keep("cum_hazard", prog.cum_hazard, np.float64), C.c_double)
        d.plans = _ptr(keep("plans", prog.plans.reshape(-1), np.int32), C.c_int32)
        d.user_records = _ptr(keep("user_records", prog.user_records, np.int32), C.c_int32)
        d.record_out = _ptr(keep("record_out", prog.record_out, np.int32), C.c_int32)
        d.bit_slot = _ptr(keep("bit_slot", prog.bit_slot, np.int32), C.c_int32)
        self.desc = d


class HostOutputs:
    """Host buffers in the ABI's shot-bit-word layout."""

    def __init__(self, prog, nshots: int):
        W = (nshots + 31) // 32
        self.W = W
        self.nshots = nshots
        self.meas = np.zeros((max(prog.num_user_records, 1), W), dtype=np.uint32)
        self.det = np.zeros((max(prog.num_detectors, 1), W), dtype=np.uint32)
        self.obs = np.zeros((max(prog.num_observables, 1), W), dtype=np.uint32)
        self.accepted = np.zeros(W, dtype=np.uint32)
        self.error = np.zeros(W, dtype=np.uint32)
        self.U, self.D, self.O = prog.num_user_records, prog.num_detectors, prog.num_observables
        o = FsSampleOut()
        o.meas = _ptr(self.meas, C.c_uint32)
        o.det = _ptr(self.det, C.c_uint32)
        o.obs = _ptr(self.obs, C.c_uint32)
        o.accepted = _ptr(self.accepted, C.c_uint32)
        o.error = _ptr(self.error, C.c_uint32)
        self.struct = o

    @staticmethod
    def unpack(words: np.ndarray, nshots: int) -> np.ndarray:
        """[rows][W] uint32 shot-bit words -> uint8 [nshots][rows]."""
        rows = words.shape[0]
        if rows == 0 or nshots == 0:
            return np.zeros((nshots, rows), dtype=np.uint8)
        b = np.unpackbits(words.astype("<u4").view(np.uint8).reshape(rows, -1),
                          axis=1, bitorder="little")[:, :nshots]
        return np.ascontiguousarray(b.T)

    def measurements(self):
        return self.unpack(self.meas[: self.U], self.nshots)

    def detectors(self):
        return self.unpack(self.det[: self.D], self.nshots)

    def observables(self):
        return self.unpack(self.obs[: self.O], self.nshots)

    def accepted_bits(self):
        return self.unpack(self.accepted[None, :], self.nshots)[:, 0]

    def error_bits(self):
        return self.unpack(self.error[None, :], self.nshots)[:, 0]


class TraceBuffers:
    """Host trace inputs/outputs (trace mode)."""

    def __init__(self, prog, nshots: int, fault_modes=None, forced=None, stop: int = -1,
                 want_state: bool = True, checkpoints=None):
        self.fault_modes = None if fault_modes is None else np.ascontiguousarray(fault_modes, dtype=np.int16)
        self.forced = None if forced is None else np.ascontiguousarray(forced, dtype=np.int8)
        if self.fault_modes is not None:
            assert self.fault_modes.shape == (nshots, prog.num_sites)
        if self.forced is not None:
            assert self.forced.shape == (nshots, prog.record_count)
        ti = FsTraceIn()
        ti.fault_modes = _ptr(self.fault_modes, C.c_int16)
        ti.forced = _ptr(self.forced, C.c_int8)
        ti.stop = stop
        self.tin = ti
        stop_eff = prog.num_instrs if stop < 0 or stop > prog.num_instrs else stop
        self.k_stop = int(prog.schedule[stop_eff - 1]) if stop_eff > 0 else 0
        self.nshots = nshots
        self.n = prog.n
        self.checkpoints = None if checkpoints is None else np.ascontiguousarray(checkpoints, dtype=np.int32)
        ncp = 0 if self.checkpoints is None else int(self.checkpoints.size)
        if ncp:
            if np.any(np.diff(self.checkpoints) <= 0) or self.checkpoints[0] < 0 or self.checkpoints[-1] > stop_eff:
                raise ValueError("checkpoints must be strictly ascending within [0, stop]")
            ti.ncheckpoints = ncp
            ti.checkpoints = _ptr(self.checkpoints, C.c_int32)
            want_state = True
        self.tout = None
        if want_state:
            n = prog.n
            self.frame_x = np.zeros((nshots, max(n, 1)), dtype=np.uint8)
            self.frame_z = np.zeros((nshots, max(n, 1)), dtype=np.uint8)
            self.gamma = np.zeros((nshots, 2), dtype=np.float64)
            self.amps = np.zeros((nshots, 1 << self.k_stop, 2), dtype=np.float64)
            self.draws = np.zeros(nshots, dtype=np.uint32)
            to = FsTraceOut()
            to.frame_x = _ptr(self.frame_x, C.c_uint8)
            to.frame_z = _ptr(self.frame_z, C.c_uint8)
            to.gamma = _ptr(self.gamma, C.c_double)
            to.amps = _ptr(self.amps, C.c_double)
            to.draws = _ptr(self.draws, C.c_uint32)
            self.records = np.zeros((nshots, max(prog.record_count, 1)), dtype=np.uint8)
            to.records = _ptr(self.records, C.c_uint8)
            if ncp:
                ks = [int(prog.schedule[c - 1]) if c > 0 else 0 for c in self.checkpoints.tolist()]
                self.cp_k = ks
                self.cp_off = np.concatenate([[0], np.cumsum([nshots << k for k in ks])]).astype(np.int64)
                self.cp_valid = np.zeros((ncp, nshots), dtype=np.uint8)
                self.cp_fx = np.zeros((ncp, nshots, max(n, 1)), dtype=np.uint8)
                self.cp_fz = np.zeros((ncp, nshots, max(n, 1)), dtype=np.uint8)
                self.cp_gamma = np.zeros((ncp, nshots, 2), dtype=np.float64)
                self.cp_amps = np.zeros((int(self.cp_off[-1]), 2), dtype=np.float64)
                to.cp_valid = _ptr(self.cp_valid, C.c_uint8)
                to.cp_frame_x = _ptr(self.cp_fx, C.c_uint8)
                to.cp_frame_z = _ptr(self.cp_fz, C.c_uint8)
                to.cp_gamma = _ptr(self.cp_gamma, C.c_double)
                to.cp_amps = _ptr(self.cp_amps, C.c_double)
            self.tout = to

    def gamma_c(self):
        return self.gamma[:, 0] + 1j * self.gamma[:, 1]

    def amps_c(self):
        return self.amps[..., 0] + 1j * self.amps[..., 1]

    def checkpoint(self, j: int) -> dict:
        """State at checkpoint j: valid [nshots], frame_x / frame_z [nshots][n], gamma [nshots],
        amps [nshots][2^k_j] (complex); entries of invalid shots are unspecified."""
        a = self.cp_amps[self.cp_off[j]:self.cp_off[j + 1]]
        a = (a[:, 0] + 1j * a[:, 1]).reshape(self.nshots, 1 << self.cp_k[j])
        return {"valid": self.cp_valid[j].astype(bool), "frame_x": self.cp_fx[j, :, :self.n],
                "frame_z": self.cp_fz[j, :, :self.n], "gamma": self.cp_gamma[j, :, 0] + 1j * self.cp_gamma[j, :, 1],
                "amps": a, "k": self.cp_k[j]}

# output formats (include/fs_sampler.h fs_format; cli.py:94-109)
FS_FMT_01 = 0
FS_FMT_BIN = 1
FS_FMT_CSV = 2
