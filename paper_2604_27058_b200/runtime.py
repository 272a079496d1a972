"""Drop-in mirror of the reference per-shot API (``framesim/runtime.py``), executed on the GPU.

Same names, arguments and error behaviour as the reference:

* ``sample(prog, shots, seed=0, workers=1, renormalize=True, stratum=None,
  keep_rejected=True)`` -> iterator of :class:`ShotRecord`  (runtime.py:777-795)
* ``sample_accumulate(prog, shots, seed=0, stratum=None)`` -> dict (runtime.py:836-867)
* ``run_shot(prog, state=None, shot=0, seed=0, forced_faults=None,
  forced_outcomes=None, weight=1.0, trace=None)`` -> ShotRecord (runtime.py:731-751)
* ``ShotState``, ``ShotRecord``, ``ShotError``, ``BRANCH_FLOOR``
* ``expectation_probe(prog, state, observable)`` (runtime.py:951-989): the active-array traversal
  runs on the GPU (``fs_probe``); the Pauli mapping uses the reference program's final tableau
* ``StratumSpec(prog, w)``, ``importance_sample(prog, stratum, shots, seed=0, workers=1,
  keep_rejected=True)`` -- stratified importance sampling (runtime.py:886-945); the per-shot
  conditional draw runs on the GPU (``fs_sample_stratum``)

``prog`` is either the reference compiler's ``BytecodeProgram`` (serialized on
first use and cached on the object) or a :class:`~.program.Program`.

Random stream: ``rng="reference"`` (default here) reproduces framesim's
SplitMix64 ``ShotRng`` draw for draw, so ``sample(prog, n, seed)`` returns the
same records as the reference; ``rng="philox"`` is the engine's native
Philox4x32-10 stream (same law, different realisation), which unlocks the
bit-sliced frame engine and is what ``bench.py`` measures.

Batched entry points (``sample_batch``) return the shot-bit-word arrays
directly; they are the throughput path (the per-shot ``ShotRecord`` objects are
a host-side convenience and cost Python time per shot).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Iterator

import numpy as np

from . import _abi
from .engine import DeviceProgram, ShotError
from .program import OP_NAMES, Program, as_program

BRANCH_FLOOR = 1e-12  # runtime.py:47
_CHUNK = 1 << 20      # shots per device call in the record iterator

__all__ = ["BRANCH_FLOOR", "FORMATS", "ShotError", "ShotRecord", "ShotState", "StratumSpec", "expectation_probe",
           "importance_sample",
           "run_shot", "sample", "sample_accumulate", "sample_batch", "sample_formatted", "write_samples",
           "Sampler", "compile_circuit"]


@dataclass(slots=True)
class ShotRecord:
    """runtime.py:59-65"""

    measurements: np.ndarray
    detectors: np.ndarray
    observables: np.ndarray
    accepted: bool
    weight: float


def _flags(rng: str, renormalize: bool = True) -> int:
    if rng not in ("reference", "philox"):
        raise ValueError(f"unknown rng {rng!r} (expected 'reference' or 'philox')")
    f = _abi.FS_RNG_SPLITMIX if rng == "reference" else _abi.FS_RNG_PHILOX
    if not renormalize:
        f |= _abi.FS_NO_RENORM
    return f


def _device_program(prog) -> DeviceProgram:
    """One resident DeviceProgram per program object (cached like the reference's closures)."""
    d = getattr(prog, "__dict__", None)
    if d is not None:
        cached = d.get("_fs_b200_device")
        if cached is not None:
            return cached
    dp = DeviceProgram(as_program(prog))
    if d is not None:
        d["_fs_b200_device"] = dp
    return dp


def compile_circuit(circuit_or_text, optimize: bool = True, postselect_detectors=()):
    """The host compiler stays the reference's (backend.py:599); re-exported for convenience."""
    try:
        from framesim.backend import compile_circuit as _cc
    except ImportError as exc:  # pragma: no cover - depends on the user's install
        raise ImportError("compile_circuit needs the reference compiler package `framesim` "
                          "(the GPU engine consumes its BytecodeProgram)") from exc
    return _cc(circuit_or_text, optimize=optimize, postselect_detectors=postselect_detectors)


class Sampler:
    """A compiled program resident on the GPU (the ``_compiled(prog)`` analogue, runtime.py:663)."""

    def __init__(self, prog, rng: str = "philox", renormalize: bool = True):
        self.prog = prog
        self.dp = _device_program(prog)
        self.flags = _flags(rng, renormalize)

    @property
    def program(self) -> Program:
        return self.dp.prog

    def sample_batch(self, shots: int, seed: int = 0, shot0: int = 0) -> dict:
        """All outputs of shots [shot0, shot0+shots) as uint8 arrays [shots, ...]."""
        if shots < 1:
            raise ValueError("shots must be >= 1")
        if shot0 % 32:
            raise ValueError("shot0 must be a multiple of 32")
        _, out, _ = self.dp.sample_host(shots, seed=seed, shot0=shot0, flags=self.flags)
        return {"measurements": out.measurements(), "detectors": out.detectors(),
                "observables": out.observables(), "accepted": out.accepted_bits().astype(bool)}

    def sample_stratum_batch(self, w: int, shots: int, seed: int = 0, shot0: int = 0) -> dict:
        """sample_batch conditioned on exactly w faults (StratumSpec.draw_forced per shot, on the GPU)."""
        if shots < 1:
            raise ValueError("shots must be >= 1")
        if shot0 % 32:
            raise ValueError("shot0 must be a multiple of 32")
        _, out = self.dp.sample_stratum_host(w, shots, seed=seed, shot0=shot0, flags=self.flags)
        return {"measurements": out.measurements(), "detectors": out.detectors(),
                "observables": out.observables(), "accepted": out.accepted_bits().astype(bool)}

    def sample_packed(self, shots: int, seed: int = 0, shot0: int = 0):
        """Raw shot-bit words (include/fs_sampler.h layout): HostOutputs."""
        _, out, _ = self.dp.sample_host(shots, seed=seed, shot0=shot0, flags=self.flags)
        return out

    def accumulate(self, shots: int, seed: int = 0) -> dict:
        acc = self.dp.accumulate(shots, seed=seed, flags=self.flags)
        acc["weight_sum"] = float(acc["accepted"])
        return acc


def sample_batch(prog, shots: int, seed: int = 0, rng: str = "reference", renormalize: bool = True) -> dict:
    return Sampler(prog, rng=rng, renormalize=renormalize).sample_batch(shots, seed=seed)


def sample(prog, shots: int, seed: int = 0, workers: int = 1, renormalize: bool = True,
           stratum=None, keep_rejected: bool = True, rng: str = "reference") -> Iterator[ShotRecord]:
    """Yield ShotRecords for shots 0..shots-1 in order (runtime.py:777-795).

    ``workers`` is accepted for signature compatibility; the GPU executes every
    shot of a chunk concurrently and the output does not depend on it.
    """
    if shots < 1:
        raise ValueError("shots must be >= 1")
    s = Sampler(prog, rng=rng, renormalize=renormalize)
    spec = _as_stratum(prog, stratum)
    return _iter_records(s, shots, seed, keep_rejected, spec)


def _iter_records(s: Sampler, shots: int, seed: int, keep_rejected: bool, spec=None):
    weight = 1.0 if spec is None else spec.weight
    for c0 in range(0, shots, _CHUNK):
        n = min(_CHUNK, shots - c0)
        if spec is None:
            b = s.sample_batch(n, seed=seed, shot0=c0)
        else:
            b = s.sample_stratum_batch(spec.w, n, seed=seed, shot0=c0)
        m, d, o, a = b["measurements"], b["detectors"], b["observables"], b["accepted"]
        for i in range(n):
            if a[i] or keep_rejected:
                yield ShotRecord(m[i], d[i], o[i], bool(a[i]), weight)


class StratumSpec:
    """Shot batch conditioned on exactly ``w`` realised faults (runtime.py:886-932).

    ``weight`` is Pr[W = w] under the Poisson-binomial law of the site probabilities (computed by
    the library exactly as the reference builds its suffix table); the per-shot conditional draw
    (``draw_forced``) runs on the GPU inside ``sample`` / ``sample_accumulate``."""

    def __init__(self, prog, w: int):
        P = as_program(prog)
        e = P.num_sites
        w = int(w)
        if w > e:
            raise ValueError(f"stratum fault count {w} exceeds {e} sites")
        if w < 0:
            raise ValueError("stratum fault count must be >= 0")
        self.w = w
        self.probs = [float(x) for x in P.site_prob]
        self.weight = _device_program(prog).stratum_weight(w)


def _as_stratum(prog, stratum):
    """None, a fault count, our StratumSpec or the reference's (anything with ``.w``)."""
    if stratum is None:
        return None
    if isinstance(stratum, StratumSpec):
        return stratum
    w = getattr(stratum, "w", stratum)
    return StratumSpec(prog, int(w))


def importance_sample(prog, stratum, shots: int, seed: int = 0, workers: int = 1, keep_rejected: bool = True,
                      rng: str = "reference"):
    """Weighted records conditioned on a fault-count stratum (runtime.py:935-945): ``stratum`` is
    a StratumSpec or a fault count w; every record carries weight Pr[W = w]."""
    return sample(prog, shots, seed=seed, workers=workers, stratum=_as_stratum(prog, stratum),
                  keep_rejected=keep_rejected, rng=rng)


def _weight_sum(weight: float, count: int) -> float:
    """The reference's running ``weight_sum += state.weight`` over accepted shots (sequential
    float additions, runtime.py:859), reproduced exactly in chunks."""
    acc = 0.0
    left = int(count)
    while left:
        m = min(left, 1 << 20)
        seq = np.empty(m + 1)
        seq[0] = acc
        seq[1:] = weight
        acc = float(np.cumsum(seq)[-1])
        left -= m
    return acc


FORMATS = {"01": _abi.FS_FMT_01, "bin": _abi.FS_FMT_BIN, "csv": _abi.FS_FMT_CSV}
_PROFILE = bool(__import__("os").environ.get("FS_FORMAT_PROFILE"))


def write_samples(prog, shots: int, out, seed: int = 0, format: str = "01", keep_rejected: bool = True,
                  stratum=None, rng: str = "reference", renormalize: bool = True, chunk: int = 1 << 20) -> int:
    """Write what ``framesim sample --format {01,bin,csv}`` writes (cli.py:94-109) to the binary
    stream ``out`` (anything with ``.write(bytes)``); returns the number of records written.

    The records are formatted on the GPU (``fs_format``), so only the final bytes cross PCIe;
    chunk i's device->host copy overlaps chunk i+1's sampling and formatting."""
    import torch

    if shots < 1:
        raise ValueError("shots must be >= 1")
    if format not in FORMATS:
        raise ValueError(f"unknown format {format!r} (expected one of {sorted(FORMATS)})")
    if chunk % 32:
        raise ValueError("chunk must be a multiple of 32")
    fmt = FORMATS[format]
    s = Sampler(prog, rng=rng, renormalize=renormalize)
    dp = s.dp
    spec = _as_stratum(prog, stratum)
    weight = 1.0 if spec is None else spec.weight
    wtext = f"{weight:.17g}"
    if format == "csv":
        out.write(b"shot,weight,bits\n")
    chunk = min(chunk, (shots + 31) // 32 * 32)
    cap = dp.format_bound(chunk, fmt, shots, wtext)
    comp, copy, slots = _format_buffers(dp, cap)
    written = 0
    pending = None  # (slot, nbytes, event)

    def flush(p):
        slot, nb, ev = p
        ev.synchronize()
        out.write(memoryview(slot["host"][:nb].numpy()))  # straight from pinned memory

    for i, c0 in enumerate(range(0, shots, chunk)):
        n = min(chunk, shots - c0)
        slot = slots[i % 2]
        if slot["copied"] is not None:
            comp.wait_event(slot["copied"])
        words = slot["words"].get(n)
        if words is None:
            with torch.cuda.stream(comp):
                words = dp.alloc_device_outputs(n)
            if len(slot["words"]) >= 4:
                slot["words"].clear()
            slot["words"][n] = words
        if _PROFILE:
            import time as _t
            _t0 = _t.perf_counter()
        if spec is None:
            dp.sample_device(n, words, seed=seed, shot0=c0, flags=s.flags, stream=comp)
        else:
            dp.sample_stratum_device(spec.w, n, words, seed=seed, shot0=c0, flags=s.flags, stream=comp)
        nb, nk = dp.format_device(n, words, fmt, keep_rejected, written, wtext, slot["dev"], stream=comp)
        if _PROFILE:
            _t1 = _t.perf_counter()
        st = int(words["status"].item())
        if st:
            from .engine import raise_for_status
            raise_for_status(st)
        ev_fmt = torch.cuda.Event()
        ev_fmt.record(comp)
        copy.wait_event(ev_fmt)
        with torch.cuda.stream(copy):
            slot["host"][:nb].copy_(slot["dev"][:nb], non_blocking=True)
        ev_cp = torch.cuda.Event()
        ev_cp.record(copy)
        slot["copied"] = ev_cp
        if pending is not None:
            flush(pending)
        if _PROFILE:
            print(f"chunk {i}: compute+format {1e3 * (_t1 - _t0):.2f} ms, to flush {1e3 * (_t.perf_counter() - _t1):.2f} ms")
        pending = (slot, nb, ev_cp)
        written += nk
    if pending is not None:
        flush(pending)
    return written


def _format_buffers(dp: DeviceProgram, cap: int):
    """Streams and two (device bytes, pinned host bytes, words) slots cached on the program:
    pinned allocations cost far more than the transfers they serve."""
    import torch

    st = dp.__dict__.setdefault("_fmt_state", {})
    if "streams" not in st:
        st["streams"] = (torch.cuda.Stream(), torch.cuda.Stream())
        st["slots"] = [{"words": {}, "dev": None, "host": None, "copied": None} for _ in range(2)]
    for slot in st["slots"]:
        if slot["dev"] is None or slot["dev"].numel() < cap:
            if slot["copied"] is not None:
                slot["copied"].synchronize()
            slot["dev"] = torch.empty(cap, dtype=torch.uint8, device="cuda")
            slot["host"] = torch.empty(cap, dtype=torch.uint8, pin_memory=True)
    return st["streams"][0], st["streams"][1], st["slots"]


def sample_formatted(prog, shots: int, seed: int = 0, format: str = "01", keep_rejected: bool = True,
                     stratum=None, rng: str = "reference", renormalize: bool = True, chunk: int = 1 << 20) -> bytes:
    """The bytes ``framesim sample --format FORMAT`` writes for these arguments (cli.py:94-109)."""
    import io

    buf = io.BytesIO()
    write_samples(prog, shots, buf, seed=seed, format=format, keep_rejected=keep_rejected, stratum=stratum,
                  rng=rng, renormalize=renormalize, chunk=chunk)
    return buf.getvalue()


def sample_accumulate(prog, shots: int, seed: int = 0, stratum=None, rng: str = "reference") -> dict:
    """Bit sums over accepted shots (runtime.py:836-867), reduced on the device."""
    if shots < 1:
        return {"shots": shots, "accepted": 0, "weight_sum": 0.0,
                "measurements": np.zeros(as_program(prog).num_user_records, np.int64),
                "detectors": np.zeros(as_program(prog).num_detectors, np.int64),
                "observables": np.zeros(as_program(prog).num_observables, np.int64)}
    spec = _as_stratum(prog, stratum)
    s = Sampler(prog, rng=rng)
    if spec is None:
        return s.accumulate(shots, seed=seed)
    acc = s.dp.accumulate_stratum(spec.w, shots, seed=seed, flags=s.flags)
    acc["weight_sum"] = _weight_sum(spec.weight, acc["accepted"])
    return acc


class ShotState:
    """Host view of one shot's factored state after ``run_shot`` (runtime.py:71-122).

    The authoritative state lives on the GPU during execution; ``run_shot``
    copies the frames, gamma, active array and record bits back here.
    """

    def __init__(self, prog, seed: int = 0, renormalize: bool = True):
        P = as_program(prog)
        self.prog = prog
        self.n = P.n
        self.k_max = P.k_max
        self.seed = seed
        self.renormalize = renormalize
        self.frame_x = np.zeros(P.n, np.uint8)
        self.frame_z = np.zeros(P.n, np.uint8)
        self.records = np.zeros(P.record_count, np.uint8)
        self.detectors = np.zeros(P.num_detectors, np.uint8)
        self.observables = np.zeros(P.num_observables, np.uint8)
        self.buf = np.zeros(1 << P.k_max, np.complex128)
        self.buf[0] = 1.0
        self.gamma = 1.0 + 0.0j
        self.k = 0
        self.weight = 1.0
        self.accepted = True
        self.draws = 0
        self.forced_faults = None
        self.forced_outcomes = None

    def active_view(self) -> np.ndarray:
        return self.buf[: 1 << self.k]


def _fault_modes(P: Program, forced_faults) -> np.ndarray | None:
    """Reference encoding (runtime.py:587-601): dict site->mode (default 0) or an array."""
    if forced_faults is None:
        return None
    if isinstance(forced_faults, dict):
        modes = np.zeros(P.num_sites, np.int16)
        for k, v in forced_faults.items():
            modes[int(k)] = int(v)
        return modes[None, :]
    arr = np.asarray(forced_faults, dtype=np.int16).reshape(1, -1)
    if arr.shape[1] != P.num_sites:
        raise ValueError("forced_faults array length must equal the number of noise sites")
    return arr


def _forced(P: Program, forced_outcomes) -> np.ndarray | None:
    if forced_outcomes is None:
        return None
    f = np.full((1, P.record_count), -1, np.int8)
    for r, b in forced_outcomes.items():
        f[0, int(r)] = int(b)
    return f


def run_shot(prog, state: ShotState | None = None, shot: int = 0, seed: int = 0, forced_faults=None,
             forced_outcomes=None, weight: float = 1.0, trace=None, rng: str = "reference") -> ShotRecord:
    """Execute one shot on the GPU; ``state`` receives its final state (runtime.py:731-751).

    ``trace(state, ins)`` is called after every instruction like the reference (a post-selected
    shot stops before the halting instruction's callback, runtime.py:749).  The states it sees
    come from the device's checkpoint dumps (fs_trace_in.checkpoints): one device call returns
    the state after every instruction, split into a few calls only when the active arrays of all
    checkpoints would exceed ``_TRACE_BYTES``.
    """
    if state is None:
        state = ShotState(prog, seed=seed)
    dp = _device_program(prog)
    P = dp.prog
    flags = _flags(rng, state.renormalize)
    fm = _fault_modes(P, forced_faults)
    fo = _forced(P, forced_outcomes)
    base = (shot // 32) * 32
    lane = shot - base
    state.forced_faults = forced_faults
    state.forced_outcomes = forced_outcomes
    state.weight = weight
    # a 1-shot call at absolute shot index `shot`: pad the word so the Philox word matches
    n = lane + 1
    fmn = None if fm is None else np.repeat(fm, n, axis=0)
    fon = None if fo is None else np.repeat(fo, n, axis=0)
    if fon is not None:
        fon[:lane] = -1

    def call(stop: int, checkpoints=None):
        st, out, tb = dp.sample_host(n, seed=state.seed, shot0=base, flags=flags, fault_modes=fmn, forced=fon,
                                     stop=stop, want_state=True, check=False, checkpoints=checkpoints)
        if st > 0 and out.error_bits()[lane]:
            from .engine import raise_for_status

            raise_for_status(st)  # errors of padding lanes are impossible (nothing forced there)
        elif st < 0:
            from .engine import raise_for_status

            raise_for_status(st)
        return out, tb

    if trace is None:
        out, tb = call(-1)
        _copy_state(state, P, out, tb, lane)
    else:
        instrs = getattr(prog, "instrs", None)
        names = {v: k for k, v in OP_NAMES.items()}
        writers = _writers(P)
        N = P.num_instrs
        out = tb = None
        i = 0
        while i < N:  # checkpoints i+1 .. j, one device call
            j, nbytes = i, 0
            while j < N and (j == i or nbytes + (16 * n << int(P.schedule[j])) <= _TRACE_BYTES):
                nbytes += 16 * n << int(P.schedule[j])
                j += 1
            out, tb = call(j, checkpoints=np.arange(i + 1, j + 1, dtype=np.int32))
            halted = False
            for c in range(i + 1, j + 1):
                cp = tb.checkpoint(c - i - 1)
                if not cp["valid"][lane]:
                    halted = True  # halted / raised before the end of instruction c-1
                    break
                _copy_checkpoint(state, P, tb, cp, lane, c, writers)
                ins = instrs[c - 1] if instrs is not None else names[int(P.instrs[c - 1, 0] & 0xFF)]
                trace(state, ins)
            if halted:
                break
            i = j
        out, tb = call(-1)
        _copy_state(state, P, out, tb, lane)
    return ShotRecord(measurements=out.measurements()[lane].copy(),
                      detectors=out.detectors()[lane].copy(),
                      observables=out.observables()[lane].copy(),
                      accepted=bool(out.accepted_bits()[lane]), weight=weight)


_TRACE_BYTES = 1 << 30  # active-array bytes of the checkpoints one traced device call returns


def _writers(P: Program) -> dict:
    """Instruction index writing each record / detector, and the observable contributions (for
    the records / detectors / observables a trace callback sees mid-program)."""
    rec_w = np.full(P.record_count, P.num_instrs, np.int64)
    det_w = np.full(P.num_detectors, P.num_instrs, np.int64)
    obs_c = []  # (instr, observable, records)
    ops = P.instrs[:, 0] & 0xFF
    for i in range(P.num_instrs):
        op = int(ops[i])
        if op in (5, 6, 7, 8):  # MeasDormantStatic/Random, MeasActive, MeasCollapse: w3 = record
            rec_w[int(P.instrs[i, 3])] = i
        elif op == 12:
            det_w[int(P.instrs[i, 1])] = i
        elif op == 13:
            off, cnt = int(P.instrs[i, 2]), int(P.instrs[i, 3])
            obs_c.append((i, int(P.instrs[i, 1]), P.reclists[off:off + cnt].astype(np.int64)))
    return {"rec": rec_w, "det": det_w, "obs": obs_c}


def _copy_checkpoint(state: ShotState, P: Program, tb, cp: dict, lane: int, c: int, writers: dict) -> None:
    """State after instructions [0, c) (device checkpoint) into ``state``."""
    state.frame_x[:] = cp["frame_x"][lane]
    state.frame_z[:] = cp["frame_z"][lane]
    state.gamma = complex(cp["gamma"][lane])
    state.k = cp["k"]
    state.buf[: 1 << cp["k"]] = cp["amps"][lane]
    final = tb.records[lane, : P.record_count]
    state.records[:] = np.where(writers["rec"] < c, final, 0)
    if P.num_detectors:
        dets = np.zeros(P.num_detectors, np.uint8)
        for d in np.flatnonzero(writers["det"] < c):
            off, cnt = _det_list(P, int(writers["det"][d]))
            dets[d] = np.bitwise_xor.reduce(final[P.reclists[off:off + cnt]]) if cnt else 0
        state.detectors[:] = dets
    if P.num_observables:
        obs = np.zeros(P.num_observables, np.uint8)
        for i, o, recs in writers["obs"]:
            if i < c and recs.size:
                obs[o] ^= np.bitwise_xor.reduce(final[recs])
        state.observables[:] = obs


def _det_list(P: Program, i: int):
    return int(P.instrs[i, 2]), int(P.instrs[i, 3])


def _copy_state(state: ShotState, P: Program, out, tb, lane: int) -> None:
    state.frame_x[:] = tb.frame_x[lane, : P.n]
    state.frame_z[:] = tb.frame_z[lane, : P.n]
    state.gamma = complex(tb.gamma_c()[lane])
    state.k = tb.k_stop
    state.buf[: 1 << tb.k_stop] = tb.amps_c()[lane]
    state.accepted = bool(out.accepted_bits()[lane])
    state.draws = int(tb.draws[lane])
    state.records[:] = tb.records[lane, : P.record_count]  # user and hidden records (ShotState.records)
    if P.num_detectors:
        state.detectors[:] = out.detectors()[lane]
    if P.num_observables:
        state.observables[:] = out.observables()[lane]


# -- expectation probe (runtime.py:951-989) --------------------------------------------------
def expectation_probe(prog, state: ShotState, observable) -> float:
    """<psi|P|psi> of the current factored state, non-collapsing (runtime.py:951-989).

    ``prog`` must be the reference compiler's BytecodeProgram: the observable is mapped through
    its ``final_tableau`` (host Pauli algebra) onto ``final_active``; the traversal of the active
    array runs on the GPU."""
    if not hasattr(prog, "final_tableau") or not hasattr(prog, "final_active"):
        raise TypeError("expectation_probe needs the reference BytecodeProgram (final_tableau, final_active)")
    if not observable.is_hermitian():
        raise ValueError("probe observable must be Hermitian")
    mapped = prog.final_tableau.heisenberg_map(observable)
    word = mapped.hermitian_word()
    return probe_mapped(state, np.asarray(word.x, np.uint8), np.asarray(word.z, np.uint8),
                        int(mapped.hermitian_sign()), list(prog.final_active))


def probe_mapped(state: ShotState, word_x, word_z, sign: int, final_active) -> float:
    """expectation_probe after the tableau mapping: Hermitian word (x, z bits over the n virtual
    qubits) with sign, on the state's frames and active array (positions = final_active)."""
    import ctypes as C

    import torch

    from . import _lib

    word_x = np.asarray(word_x, np.uint8)
    word_z = np.asarray(word_z, np.uint8)
    par = (int(np.count_nonzero(word_x & state.frame_z)) + int(np.count_nonzero(word_z & state.frame_x))) & 1
    active_pos = {int(v): p for p, v in enumerate(final_active)}
    xm = zm = 0
    ycount = 0
    for j in np.flatnonzero(word_x | word_z):
        j = int(j)
        if j not in active_pos:
            if word_x[j]:
                return 0.0
            continue
        p = active_pos[j]
        if word_x[j]:
            xm |= 1 << p
        if word_z[j]:
            zm |= 1 << p
        if word_x[j] and word_z[j]:
            ycount += 1
    amps = np.ascontiguousarray(state.active_view())
    dev = torch.from_numpy(amps.view(np.float64)).to("cuda")
    out = (C.c_double * 2)()
    s = torch.cuda.current_stream()
    rc = _lib.lib().fs_probe(C.c_void_p(dev.data_ptr()), int(state.k), xm, zm, ycount, out, C.c_void_p(s.cuda_stream))
    if rc != 0:
        raise ValueError(_lib.last_error())
    val = out[0] / out[1]
    return sign * (-1.0 if par else 1.0) * val
