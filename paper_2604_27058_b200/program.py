"""Flat, device-ready encoding of a compiled bytecode program.

The reference compiler (``framesim.backend.compile_circuit``,
``/root/reference/pkg/src/framesim/backend.py:599``) produces an immutable
``BytecodeProgram`` (``backend.py:254-269``) holding 15 frozen instruction
dataclasses (``backend.py:107-241``).  The reference VM specialises each one
into a Python closure (``runtime.py:644-669``).  Here the same program is
flattened once, on the host, into plain arrays that the C-ABI
(``include/fs_sampler.h``) copies to the GPU:

* ``instrs``      int32[N][8]  opcode word + 7 operands (layout in fs_sampler.h)
* ``fparams``     float64[]    precomputed phases / 2x2 unitaries (same cmath
                               expressions as the reference closures, so the
                               constants are bit-identical)
* ``gates``       uint32[]     packed frame gates ``g<<28 | a<<14 | b``
* ``paulis``      uint32[]     sparse Pauli masks ``q<<1 | is_z``
* ``reclists``    int32[]      detector / observable record lists
* site tables, ``cum_hazard``, per-block hazard plans (``runtime.py:710-725``)
* record routing: output column of every user record, and an on-chip "slot"
  for every bit (record or detector) that a later instruction reads.

Nothing here executes a shot; it is the boundary data format.
"""
from __future__ import annotations

import cmath
import io
import math
from dataclasses import dataclass, field

import numpy as np

# opcode numbering: must match include/fs_sampler.h
OP_FRAME = 0
OP_ARRAY_GATE = 1
OP_EXPAND = 2
OP_GAMMA_ROT = 3
OP_ARRAY_ROT = 4
OP_MEAS_DSTATIC = 5
OP_MEAS_DRANDOM = 6
OP_MEAS_ACTIVE = 7
OP_MEAS_COLLAPSE = 8
OP_RETIRE = 9
OP_COND_FRAME = 10
OP_NOISE = 11
OP_DETECTOR = 12
OP_OBSERVABLE = 13
OP_POSTSELECT = 14

OP_NAMES = {
    "FrameGates": OP_FRAME, "ArrayGate": OP_ARRAY_GATE, "Expand": OP_EXPAND,
    "GammaRot": OP_GAMMA_ROT, "ArrayRot": OP_ARRAY_ROT,
    "MeasDormantStatic": OP_MEAS_DSTATIC, "MeasDormantRandom": OP_MEAS_DRANDOM,
    "MeasActive": OP_MEAS_ACTIVE, "MeasCollapse": OP_MEAS_COLLAPSE,
    "Retire": OP_RETIRE, "CondFrame": OP_COND_FRAME, "NoiseBlock": OP_NOISE,
    "DetectorIns": OP_DETECTOR, "ObservableIns": OP_OBSERVABLE,
    "PostSelectIns": OP_POSTSELECT,
}

G_H, G_S, G_SDAG, G_CX, G_CZ, G_SWAP = range(6)
_GATE_CODE = {"H": G_H, "S": G_S, "S_DAG": G_SDAG, "CX": G_CX, "CZ": G_CZ, "SWAP": G_SWAP}
_NOOP_GATES = ("X", "Y", "Z")  # conjugation by X/Y/Z never moves frame bits (runtime.py:149)

MAX_QUBITS = 1 << 14
INV_SQRT2 = 1.0 / math.sqrt(2.0)  # runtime.py:46

ARRAY_OPS = (OP_ARRAY_GATE, OP_EXPAND, OP_ARRAY_ROT, OP_MEAS_ACTIVE, OP_MEAS_COLLAPSE, OP_RETIRE)


class ProgramError(ValueError):
    pass


def _pack_gate(g: int, a: int, b: int | None) -> int:
    return (g << 28) | (a << 14) | (0 if b is None else b)


@dataclass
class Program:
    """Serialized BytecodeProgram (see module docstring)."""

    n: int
    k_max: int
    record_count: int
    num_detectors: int
    num_observables: int
    instrs: np.ndarray          # int32 [N, 8]
    schedule: np.ndarray        # int32 [N]  active dimension after each instruction
    fparams: np.ndarray         # float64
    gates: np.ndarray           # uint32
    paulis: np.ndarray          # uint32
    reclists: np.ndarray        # int32
    site_prob: np.ndarray       # float64 [E]
    site_case_off: np.ndarray   # int32 [E+1]
    case_cum: np.ndarray        # float64 [C]
    case_pauli_off: np.ndarray  # int32 [C+1]
    cum_hazard: np.ndarray      # float64 [E+1]
    plans: np.ndarray           # int32 [P, 2]  (a, b) segment or (-1, s) certain site
    user_records: np.ndarray    # int32 [U]
    record_out: np.ndarray      # int32 [R]  user column or -1 (hidden)
    bit_slot: np.ndarray        # int32 [R + D]  on-chip slot of a record/detector bit, -1 if never read
    num_slots: int
    name: str = ""
    meta: dict = field(default_factory=dict)

    # -- derived ---------------------------------------------------------------
    @property
    def num_instrs(self) -> int:
        return int(self.instrs.shape[0])

    @property
    def num_sites(self) -> int:
        return int(self.site_prob.shape[0])

    @property
    def num_user_records(self) -> int:
        return int(self.user_records.shape[0])

    @property
    def has_postselect(self) -> bool:
        return bool(np.any((self.instrs[:, 0] & 0xFF) == OP_POSTSELECT))

    @property
    def frame_only(self) -> bool:
        return self.k_max == 0

    def opcode_counts(self) -> dict:
        inv = {v: k for k, v in OP_NAMES.items()}
        ops, cnt = np.unique(self.instrs[:, 0] & 0xFF, return_counts=True)
        return {inv[int(o)]: int(c) for o, c in zip(ops, cnt)}

    def work(self) -> int:
        """W = sum of array sweep sizes (reference ``plan_metrics``, backend.py:498-506)."""
        ops = self.instrs[:, 0] & 0xFF
        w = 0
        for i in range(self.num_instrs):
            if int(ops[i]) in ARRAY_OPS:
                w += 1 << int(self.instrs[i, 6])
        return w

    def output_bits(self) -> int:
        return self.num_user_records + self.num_detectors + self.num_observables

    # -- persistence -------------------------------------------------------------
    _ARRAYS = ("instrs", "schedule", "fparams", "gates", "paulis", "reclists",
               "site_prob", "site_case_off", "case_cum", "case_pauli_off",
               "cum_hazard", "plans", "user_records", "record_out", "bit_slot")
    _SCALARS = ("n", "k_max", "record_count", "num_detectors", "num_observables",
                "num_slots")

    def to_npz_bytes(self) -> bytes:
        buf = io.BytesIO()
        payload = {k: getattr(self, k) for k in self._ARRAYS}
        payload["scalars"] = np.array([getattr(self, k) for k in self._SCALARS], dtype=np.int64)
        payload["name"] = np.array(self.name)
        payload["meta"] = np.array(repr(self.meta))
        np.savez_compressed(buf, **payload)
        return buf.getvalue()

    def save(self, path) -> None:
        with open(path, "wb") as f:
            f.write(self.to_npz_bytes())

    @classmethod
    def load(cls, path_or_file) -> "Program":
        import ast

        with np.load(path_or_file, allow_pickle=False) as z:
            sc = z["scalars"].tolist()
            kw = {k: int(v) for k, v in zip(cls._SCALARS, sc)}
            for k in cls._ARRAYS:
                kw[k] = z[k]
            kw["name"] = str(z["name"])
            kw["meta"] = ast.literal_eval(str(z["meta"]))
        return cls(**kw)


def _bits_to_paulis(xmask, zmask) -> list[int]:
    out = []
    xs = np.flatnonzero(np.asarray(xmask, dtype=np.uint8))
    zs = np.flatnonzero(np.asarray(zmask, dtype=np.uint8))
    for q in xs:
        out.append(int(q) << 1)
    for q in zs:
        out.append((int(q) << 1) | 1)
    return out


def _c(v: complex) -> list[float]:
    v = complex(v)
    return [v.real, v.imag]


def serialize(prog, name: str = "", meta: dict | None = None) -> Program:
    """Flatten a reference ``BytecodeProgram`` (duck-typed) into a :class:`Program`."""
    n = int(prog.n)
    if n >= MAX_QUBITS:
        raise ProgramError(f"n={n} exceeds the encoding limit {MAX_QUBITS - 1}")
    R = int(prog.record_count)
    D = int(prog.num_detectors)
    instrs: list[list[int]] = []
    fparams: list[float] = []
    gates: list[int] = []
    paulis: list[int] = []
    reclists: list[int] = []
    plans: list[tuple[int, int]] = []
    # bit reads for slot allocation: bit id -> (first write instr, last read instr)
    first_write: dict[int, int] = {}
    last_read: dict[int, int] = {}

    def wrote(bit: int, i: int) -> None:
        first_write.setdefault(bit, i)

    def read(bit: int, i: int) -> None:
        last_read[bit] = i

    def fp(vals) -> int:
        off = len(fparams)
        fparams.extend(float(v) for v in vals)
        return off

    sites = prog.sites
    n_coins = 0
    for i, ins in enumerate(prog.instrs):
        kind = type(ins).__name__
        if kind not in OP_NAMES:
            raise ProgramError(f"unknown instruction {kind}")
        op = OP_NAMES[kind]
        w = [op, 0, 0, 0, 0, 0, 0, 0]
        if op == OP_FRAME:
            off = len(gates)
            for g, a, b in ins.gates:
                if g in _NOOP_GATES:
                    continue
                gates.append(_pack_gate(_GATE_CODE[g], int(a), None if b is None else int(b)))
            w[1], w[2] = off, len(gates) - off
        elif op == OP_ARRAY_GATE:
            w[1] = _GATE_CODE[ins.gate]
            w[2] = int(ins.va)
            w[3] = -1 if ins.vb is None else int(ins.vb)
            w[4] = int(ins.axa)
            w[5] = -1 if ins.axb is None else int(ins.axb)
            w[6] = int(ins.size).bit_length() - 1
        elif op == OP_EXPAND:
            # phases[parity] = (ph0, ph1), exactly as runtime.py:242-247
            if ins.fused:
                e0 = cmath.exp(-1j * ins.angle) * INV_SQRT2
                e1 = cmath.exp(1j * ins.angle) * INV_SQRT2
                ph = ((e0, e1), (e1, e0))
            else:
                ph = ((INV_SQRT2, INV_SQRT2),) * 2
            w[1] = int(ins.virt)
            w[2] = int(ins.axis)
            w[5] = fp(_c(ph[0][0]) + _c(ph[0][1]) + _c(ph[1][0]) + _c(ph[1][1]))
            w[6] = int(ins.size).bit_length() - 1          # k before expansion
        elif op == OP_GAMMA_ROT:
            ph = (cmath.exp(-1j * ins.angle), cmath.exp(1j * ins.angle))  # runtime.py:268
            w[1] = int(ins.virt)
            w[5] = fp(_c(ph[0]) + _c(ph[1]))
        elif op == OP_ARRAY_ROT:
            e0 = cmath.exp(-1j * ins.angle)                 # runtime.py:278-280
            e1 = e0.conjugate()
            w[1] = int(ins.virt)
            w[2] = int(ins.axis)
            w[5] = fp(_c(e0) + _c(e1))
            w[6] = int(ins.size).bit_length() - 1
        elif op in (OP_MEAS_DSTATIC, OP_MEAS_DRANDOM):
            w[0] |= int(ins.flip) << 8
            w[1] = int(ins.virt)
            w[3] = int(ins.record)
            if op == OP_MEAS_DRANDOM:  # coin ordinal: 4 coin words per Philox block
                w[2] = n_coins
                n_coins += 1
            wrote(int(ins.record), i)
        elif op in (OP_MEAS_ACTIVE, OP_MEAS_COLLAPSE):
            w[0] |= int(ins.flip) << 8
            w[1] = int(ins.virt)
            w[2] = int(ins.axis)
            w[3] = int(ins.record)
            w[6] = int(ins.size).bit_length() - 1
            wrote(int(ins.record), i)
            if op == OP_MEAS_COLLAPSE:
                (u00, u01), (u10, u11) = ins.u
                w[5] = fp(_c(u00) + _c(u01) + _c(u10) + _c(u11))
                off = len(gates)
                for g, q, _ in ins.pre_gates:
                    gates.append(_pack_gate(_GATE_CODE[g], int(q), None))
                w[4] = (off << 8) | (len(gates) - off)
                if len(gates) - off > 255:
                    raise ProgramError("too many collapse pre-gates")
        elif op == OP_RETIRE:
            w[1] = int(ins.virt)
            w[2] = int(ins.axis)
            w[6] = int(ins.size).bit_length() - 1
        elif op == OP_COND_FRAME:
            off = len(paulis)
            paulis.extend(_bits_to_paulis(ins.xmask, ins.zmask))
            w[1], w[2] = off, len(paulis) - off
            w[3] = int(ins.record)
            read(int(ins.record), i)
        elif op == OP_NOISE:
            lo, hi = int(ins.lo), int(ins.hi)
            off = len(plans)
            start = lo
            for s in range(lo, hi):                         # runtime.py:710-725
                if sites[s].prob >= 1.0:
                    if start < s:
                        plans.append((start, s))
                    plans.append((-1, s))
                    start = s + 1
            if start < hi:
                plans.append((start, hi))
            w[1], w[2] = lo, hi
            w[3], w[4] = off, len(plans) - off
        elif op in (OP_DETECTOR, OP_OBSERVABLE):
            off = len(reclists)
            recs = [int(r) for r in ins.records]
            reclists.extend(recs)
            for r in recs:
                read(r, i)
            w[1] = int(ins.index)
            w[2], w[3] = off, len(recs)
            if op == OP_DETECTOR:
                wrote(R + int(ins.index), i)
        elif op == OP_POSTSELECT:
            is_det = ins.kind == "detector"
            w[1] = 0 if is_det else 1
            w[2] = int(ins.ref)
            w[3] = int(ins.required)
            read((R + int(ins.ref)) if is_det else int(ins.ref), i)
        instrs.append(w)

    # site tables
    E = len(sites)
    site_prob = np.array([float(s.prob) for s in sites], dtype=np.float64)
    site_case_off = [0]
    case_cum: list[float] = []
    case_pauli_off = [len(paulis)]   # absolute offsets into `paulis`
    for s in sites:
        for c in range(len(s.case_cum)):
            case_cum.append(float(s.case_cum[c]))
            paulis_c = _bits_to_paulis(s.case_x[c], s.case_z[c])
            paulis.extend(paulis_c)
            case_pauli_off.append(len(paulis))
        site_case_off.append(len(case_cum))
    cpo = np.array(case_pauli_off, dtype=np.int32)

    # slot allocation: interval colouring of bits that are read after written
    intervals = []
    for bit, last in last_read.items():
        if bit not in first_write:
            raise ProgramError(f"bit {bit} read before it is written")
        intervals.append((first_write[bit], last, bit))
    intervals.sort()
    bit_slot = np.full(R + D, -1, dtype=np.int32)
    free: list[int] = []
    active: list[tuple[int, int]] = []  # (last_read, slot)
    nslots = 0
    import heapq
    for start, end, bit in intervals:
        while active and active[0][0] < start:
            _, s = heapq.heappop(active)
            free.append(s)
        if free:
            slot = free.pop()
        else:
            slot = nslots
            nslots += 1
        bit_slot[bit] = slot
        heapq.heappush(active, (end, slot))

    user = np.array(prog.user_records, dtype=np.int32)
    record_out = np.full(R, -1, dtype=np.int32)
    for j, r in enumerate(user.tolist()):
        record_out[r] = j

    ins_arr = np.array(instrs, dtype=np.int32).reshape(-1, 8)
    sched = np.array(prog.active_schedule, dtype=np.int32)
    if sched.shape[0] != ins_arr.shape[0]:
        raise ProgramError("schedule length mismatch")
    m = dict(meta or {})
    return Program(
        n=n, k_max=int(prog.k_max), record_count=R, num_detectors=D,
        num_observables=int(prog.num_observables),
        instrs=ins_arr, schedule=sched,
        fparams=np.array(fparams, dtype=np.float64),
        gates=np.array(gates, dtype=np.uint32),
        paulis=np.array(paulis, dtype=np.uint32),
        reclists=np.array(reclists, dtype=np.int32),
        site_prob=site_prob,
        site_case_off=np.array(site_case_off, dtype=np.int32),
        case_cum=np.array(case_cum, dtype=np.float64),
        case_pauli_off=cpo,
        cum_hazard=np.array([float(x) for x in prog.cum_hazard], dtype=np.float64),
        plans=np.array(plans, dtype=np.int32).reshape(-1, 2),
        user_records=user, record_out=record_out, bit_slot=bit_slot,
        num_slots=int(nslots), name=name, meta=m)


def as_program(prog) -> Program:
    """Accept a serialized :class:`Program` or a reference ``BytecodeProgram``."""
    if isinstance(prog, Program):
        return prog
    cached = getattr(prog, "__dict__", {}).get("_fs_b200_program")
    if cached is not None:
        return cached
    p = serialize(prog)
    try:
        # underscore caches are stripped by BytecodeProgram.__getstate__ (backend.py:280-285)
        prog.__dict__["_fs_b200_program"] = p
    except (AttributeError, TypeError):
        pass
    return p
