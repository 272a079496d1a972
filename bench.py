#!/usr/bin/env python
"""Benchmark: shots/s of the B200 sampling engine on the BASELINE.json configurations.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

A "step" is one pass of the hot path over one batch: ``fs_sample`` of the
config's full shot count (config 1: 1e7 shots of the d=5 r=5 surface-code
memory) with the compiled program resident in HBM.  ``value`` is whole-job
shots/s from CUDA-event device time of the K timed steps (L2 flushed between
steps by writing a 256 MiB buffer, outside the events); ``e2e`` is the same
metric through the C-ABI host call ``fs_sample_host`` into pinned host buffers
(device->host copy of every output bit inside the timed region).

``--impl reference`` times the reference algorithm on the host CPU cores: the
oracle restatement (oracle/fs_oracle.c, the reference VM with its own
SplitMix64 stream, bit-exact with framesim.runtime per tests/test_oracle_golden.py)
on all host cores, each step a bounded sample of the same workload.

Multi-GPU (torchrun): weak scaling, every rank samples its own shot range
(shot0 = rank * shots) with no collective on the data path; max-over-ranks time.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

from paper_2604_27058_b200.configs import CONFIGS  # noqa: E402
from paper_2604_27058_b200.program import Program  # noqa: E402

PROGS = ROOT / "paper_2604_27058_b200" / "programs"
METRIC = "shots/sec on 1 B200 vs peak active dim k; % of HBM/on-chip roofline"


def peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons DURING the timed region (B200_PROFILING.md)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}", "--format=csv,noheader",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1].split()[0]))
                smax = float(f[2].split()[0])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- CPU reference
def _oracle_worker(args):
    path, seed, shot0, nshots = args
    import oracle
    from paper_2604_27058_b200._abi import FS_RNG_SPLITMIX

    P = Program.load(path)
    t0 = time.perf_counter()
    st, _ = oracle.accumulate(P, nshots, seed=seed, shot0=shot0, flags=FS_RNG_SPLITMIX)
    return time.perf_counter() - t0, st


def cpu_reference_rate(cfg: int, target_s: float = 8.0, cores: int | None = None) -> dict:
    """Reference algorithm (oracle port, reference SplitMix64 stream) on all host cores."""
    import multiprocessing as mp

    import oracle

    oracle.build()
    path = PROGS / f"c{cfg}.npz"
    cores = cores or os.cpu_count() or 1
    if target_s <= 0.0:  # one 32-shot word per core (config 3: seconds per shot)
        per_core = 32 if Program.load(path).k_max < 16 else 1
    else:
        # calibrate on one core
        probe = 256
        while True:
            dt, _ = _oracle_worker((path, 1, 0, probe))
            if dt > 0.5 or probe >= 1 << 20:
                break
            probe *= 4
        rate1 = probe / dt
        per_core = max(32, int(rate1 * target_s) // 32 * 32)
    stride = (per_core + 31) // 32 * 32  # shot ranges start on 32-shot words
    jobs = [(path, 7, c * stride, per_core) for c in range(cores)]
    t0 = time.perf_counter()
    with mp.get_context("fork").Pool(cores) as pool:
        res = pool.map(_oracle_worker, jobs)
    wall = time.perf_counter() - t0
    shots = per_core * cores
    return {"value": shots / wall, "unit": "shots/s", "cores": cores, "kind": "port",
            "sample": f"{shots} shots of config {cfg} ({per_core}/core, reference SplitMix64 stream, "
                      f"oracle/fs_oracle.c); {wall:.1f}s wall"}


def run_reference_arm(args, rank: int, world: int) -> None:
    if rank != 0:
        return
    cfg = args.config
    vals = []
    for _ in range(args.warmup if args.warmup < 2 else 1):
        cpu_reference_rate(cfg, target_s=1.0)
    for _ in range(args.steps):
        vals.append(cpu_reference_rate(cfg, target_s=max(2.0, 20.0 / max(args.steps, 1))))
    v = float(np.median([x["value"] for x in vals]))
    base = vals[-1]
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "shots/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": None, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(cfg),
        "cpu_baseline": {"value": v, "unit": "shots/s", "cores": base["cores"], "kind": base["kind"],
                         "sample": base["sample"]},
        "e2e": {"value": v, "unit": "shots/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- GPU arm
def workload_config(cfg: int) -> dict:
    P = Program.load(PROGS / f"c{cfg}.npz")
    return {"workload": f"config{cfg}:{CONFIGS[cfg]['name']}", "desc": CONFIGS[cfg]["desc"],
            "shots_per_step": CONFIGS[cfg]["shots"], "n_qubits": P.n, "k_max": P.k_max,
            "instructions": P.num_instrs, "noise_sites": P.num_sites,
            "output_bits_per_shot": P.output_bits(),
            "l2": "flushed between steps (256 MiB write, outside the events)",
            "parallelism": "replicas (shot ranges), no collective"}


KERNEL_NAME = {"frame": "fs_aff_frame (affine frame kernel: fault-effect row tables, warp-cooperative noise stream)",
               "general": "fs_jit_general (program-specialised general kernel, NVRTC)",
               "segmented": "fs_seg_<b> (program-specialised post-select segments: lane / warp / CTA per shot, NVRTC)",
               "hbm": "fs_pass_<i> (program-specialised fused tile passes, NVRTC)"}


def algorithmic_bytes_per_shot(P: Program) -> float:
    """Output-bound unit: user records + detectors + observables, bit-packed."""
    return P.output_bits() / 8.0


def time_gpu_config(cfg: int, steps: int, warmup: int, rank: int, shots: int | None = None,
                    warm_shots: int | None = None) -> dict:
    import ctypes as C

    import torch

    from paper_2604_27058_b200.engine import DeviceProgram

    P = Program.load(PROGS / f"c{cfg}.npz")
    dp = DeviceProgram(P)
    shots = shots or CONFIGS[cfg]["shots"]
    shot0 = rank * ((shots + 31) // 32 * 32)
    out = dp.alloc_device_outputs(shots)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream()
    for w in range(warmup):
        dp.sample_device(warm_shots or shots, out, seed=1000 + w, shot0=shot0)
    torch.cuda.synchronize()
    L = dp._lib
    L.fs_debug_launches.restype = C.c_uint64
    L.fs_debug_launches.argtypes = [C.c_void_p]
    L.fs_debug_kernel_timer.argtypes = [C.c_void_p, C.c_int]
    L.fs_debug_kernel_time.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_int64)]
    L.fs_debug_kernel_timer(dp._h, 1)  # events around the dominant kernel's launches
    n0 = L.fs_debug_launches(dp._h)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for k in range(steps):
        flush.fill_(k & 0xFF)
        ev[k][0].record(stream)
        dp.sample_device(shots, out, seed=k, shot0=shot0)
        ev[k][1].record(stream)
    torch.cuda.synchronize()
    launches = int(L.fs_debug_launches(dp._h) - n0)
    kms, kn = C.c_double(0.0), C.c_int64(0)
    L.fs_debug_kernel_time(dp._h, C.byref(kms), C.byref(kn))
    L.fs_debug_kernel_timer(dp._h, 0)
    ms = [a.elapsed_time(b) for a, b in ev]
    st = int(out["status"].item())
    return {"P": P, "dp": dp, "shots": shots, "shot0": shot0, "ms": ms, "status": st,
            "engine": dp.engine(0), "out": out, "launches": launches,
            "kernel_ms": float(kms.value), "kernel_launches": int(kn.value)}


def fp64_peak() -> float:
    """Measured FP64 FMA throughput (TFLOP/s) of this device: the on-chip roofline denominator."""
    import ctypes as C

    from paper_2604_27058_b200 import _lib

    v = C.c_double(0.0)
    L = _lib.lib()
    L.fs_debug_fp64_peak.argtypes = [C.POINTER(C.c_double)]
    L.fs_debug_fp64_peak(C.byref(v))
    return float(v.value)


def segment_work(P: Program) -> list[tuple[int, int, int]]:
    """(begin, end, W) of the post-select segments (the whole program if none)."""
    ops = P.instrs[:, 0] & 0xFF
    bounds = [0] + [int(i) + 1 for i in np.nonzero(ops == 14)[0] if i + 1 < P.num_instrs] + [P.num_instrs]
    arr = (1, 2, 4, 7, 8, 9)
    out = []
    for b, e in zip(bounds[:-1], bounds[1:]):
        w = sum(1 << int(P.instrs[i, 6]) for i in range(b, e) if int(ops[i]) in arr)
        out.append((b, e, w))
    return out


def extra_config(c: int, fp64_tflops: float, cpu: bool = True) -> dict:
    """Side measurement of another BASELINE config: device-timed shots/s with its own
    roofline, the same metric end to end through fs_sample_host (D2H inside the timed region), and
    the reference algorithm on the host cores (oracle port, all cores, bounded sample)."""
    import ctypes as C

    steps = 1 if c == 3 else 3
    rc = time_gpu_config(c, steps, 1, 0)
    P, shots = rc["P"], rc["shots"]
    ms = float(np.mean(rc["ms"]))
    rate = shots / (ms / 1e3)
    engine = rc["engine"]
    if engine == "general" and P.has_postselect:
        engine = "segmented"
    d = {"shots_per_s": rate, "ms_per_step": ms, "shots": shots, "k_max": P.k_max, "engine": engine,
         "kernel": KERNEL_NAME.get(engine, engine), "status": rc["status"]}
    e2e_steps = 1 if c in (3, 4) else 2
    e = time_e2e(rc["dp"], P, shots, 0, e2e_steps)
    d["e2e"] = {"value": shots * e2e_steps / e["seconds"], "unit": "shots/s",
                "h2d_bytes_per_step": e["h2d_bytes_per_step"], "d2h_bytes_per_step": e["d2h_bytes_per_step"]}
    if cpu:
        d["cpu_baseline"] = cpu_reference_rate(c, target_s=3.0 if c != 3 else 0.0)
        d["vs_cpu"] = {"device": rate / d["cpu_baseline"]["value"],
                       "e2e": d["e2e"]["value"] / d["cpu_baseline"]["value"]}
    d["gpu_launches_per_step"] = rc["launches"] / steps
    d["dominant_kernel_share"] = rc["kernel_ms"] / (ms * steps)
    if c == 3:  # fused tile passes: each reads + writes the live array of every shot once
        bits = (C.c_int32 * 4096)()
        L = rc["dp"]._lib
        L.fs_debug_hbm_pass_bits.restype = C.c_int64
        L.fs_debug_hbm_pass_bits.argtypes = [C.c_void_p, C.POINTER(C.c_int32), C.c_int64]
        npass = L.fs_debug_hbm_pass_bits(rc["dp"]._h, bits, 4096)
        pass_bytes = sum(32.0 * (1 << bits[i]) for i in range(npass)) * shots * steps
        ach = pass_bytes / (rc["kernel_ms"] / 1e3) / 1e9
        pk = peaks()["hbm_gbs"]
        W = P.work()
        d["roofline"] = {"bound": "hbm", "unit": "GB/s", "achieved": ach, "peak": pk, "frac": ach / pk,
                         "kernel": KERNEL_NAME["hbm"], "passes": npass,
                         "bytes_per_shot": pass_bytes / (shots * steps),
                         "unfused_algorithmic_bytes_per_shot": 32.0 * W,
                         "note": "bytes = one complex128 read + write of the live array per fused pass; "
                                 "the reference's per-instruction sweeps would move 32*W bytes per shot"}
    else:  # on-chip bound: 8 FP64 flop per element-sweep of the executed instructions
        segs = segment_work(P)
        if len(segs) > 1:
            L = rc["dp"]._lib
            L.fs_debug_seg_counts.argtypes = [C.c_void_p, C.POINTER(C.c_uint32), C.c_int]
            buf = (C.c_uint32 * 4096)()
            n = L.fs_debug_seg_counts(rc["dp"]._h, buf, 4096)
            counts = list(buf[:n])
            # counts: per chunk, [n_in(seg0), n_out(seg0)=n_in(seg1), ...]
            wexec, i = 0.0, 0
            while i < len(counts):
                chunk = counts[i:i + len(segs)]
                for (b, e, w), nin in zip(segs, chunk):
                    wexec += w * nin
                i += len(segs)
            w_exec = wexec / shots
        else:
            w_exec = float(segs[0][2])
        ach = 8.0 * w_exec * shots * steps / (rc["kernel_ms"] / 1e3) / 1e12
        d["roofline"] = {"bound": "fp64", "unit": "TFLOP/s", "achieved": ach, "peak": fp64_tflops,
                         "frac": ach / fp64_tflops if fp64_tflops else None,
                         "w_exec_per_shot": w_exec, "flop_per_shot": 8.0 * w_exec,
                         "peak_source": "measured FP64 FMA microbenchmark (fs_debug_fp64_peak)"}
    del rc
    return d


def time_e2e(dp, P, shots: int, shot0: int, steps: int) -> dict:
    """fs_sample_host into pinned host buffers: D2H of every output word inside the timed region."""
    import ctypes as C

    import torch

    from paper_2604_27058_b200._abi import FsSampleOut, vptr

    W = (shots + 31) // 32
    rows = {"meas": max(P.num_user_records, 1), "det": max(P.num_detectors, 1),
            "obs": max(P.num_observables, 1)}
    host = {k: torch.empty((r, W), dtype=torch.int32, pin_memory=True) for k, r in rows.items()}
    host["accepted"] = torch.empty(W, dtype=torch.int32, pin_memory=True)
    host["error"] = torch.empty(W, dtype=torch.int32, pin_memory=True)
    status = torch.zeros(1, dtype=torch.int32, pin_memory=True)
    o = FsSampleOut()
    for k in ("meas", "det", "obs", "accepted", "error"):
        setattr(o, k, vptr(host[k].data_ptr(), C.c_uint32))
    o.status = vptr(status.data_ptr(), C.c_int32)
    lib = dp._lib
    d2h = 4 * W * (P.num_user_records + P.num_detectors + P.num_observables + 2) + 4
    lib.fs_sample_host(dp._h, 5, shot0, shots, 0, None, C.byref(o), None)  # warm (staging alloc)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k in range(steps):
        rc = lib.fs_sample_host(dp._h, k, shot0, shots, 0, None, C.byref(o), None)
        if rc != 0:
            raise RuntimeError(f"fs_sample_host rc={rc}")
    dt = time.perf_counter() - t0
    return {"seconds": dt, "d2h_bytes_per_step": d2h, "h2d_bytes_per_step": 0}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=1, help="BASELINE.json config index (headline: 1)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-extra", action="store_true", help="skip the per-config side table")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch.distributed as dist_

        dist = dist_
        backend = "gloo" if args.impl == "reference" else "nccl"
        if backend == "nccl":
            import torch

            torch.cuda.set_device(local)
        dist.init_process_group(backend=backend)

    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        if dist:
            dist.barrier()
            dist.destroy_process_group()
        return

    import torch

    torch.cuda.set_device(local)
    from paper_2604_27058_b200 import _lib

    _lib.lib()  # fail loudly if the engine is missing
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    clk = ClockSampler(local).start()
    r = time_gpu_config(args.config, args.steps, args.warmup, rank)
    torch.cuda.synchronize()
    clocks = clk.stop()
    if r["status"] != 0:
        raise SystemExit(f"engine reported shot errors: status={r['status']}")
    dev_s = sum(r["ms"]) / 1e3
    if dist:
        t = torch.tensor([dev_s], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dev_s = float(t.item())
    P = r["P"]
    shots = r["shots"]
    total_shots = shots * args.steps * world
    value = total_shots / dev_s
    avg_ms = dev_s / args.steps * 1e3
    pk = peaks()
    # dominant kernel: its own launches, timed with CUDA events on the launching stream
    kern_ms = r["kernel_ms"] / max(r["kernel_launches"], 1)
    bytes_per_launch = algorithmic_bytes_per_shot(P) * shots * args.steps / max(r["kernel_launches"], 1)
    achieved = bytes_per_launch / (kern_ms / 1e3) / 1e9
    traffic = None
    tf = ROOT / "profiles" / "ncu_traffic.json"
    if tf.exists():
        try:
            traffic = json.loads(tf.read_text()).get(f"config{args.config}")
        except (ValueError, OSError):
            traffic = None

    e2e = time_e2e(r["dp"], P, shots, r["shot0"], max(2, min(args.steps, 5)))
    e2e_steps = max(2, min(args.steps, 5))
    e2e_s = e2e["seconds"]
    if dist:
        t = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_value = shots * e2e_steps * world / e2e_s

    extra = {}
    if not args.no_extra and rank == 0:
        fp64 = fp64_peak()
        for c in (0, 2, 3, 4):
            if c == args.config:
                continue
            try:
                extra[f"config{c}"] = extra_config(c, fp64)
            except Exception as exc:  # report, don't mask
                extra[f"config{c}"] = {"error": repr(exc)}
        extra["fp64_peak_tflops_measured"] = fp64
    cpu = None
    if not args.no_cpu and rank == 0 and world == 1:
        cpu = cpu_reference_rate(args.config, target_s=8.0)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "shots/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": avg_ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u32 (bit-sliced frames) / f64", "data": "synthetic",
            "config": workload_config(args.config),
            "engine": r["engine"],
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
                         "frac": achieved / pk["hbm_gbs"], "traffic": traffic,
                         "algorithmic_bytes_per_launch": bytes_per_launch,
                         "kernel": KERNEL_NAME.get(r["engine"], r["engine"]),
                         "kernel_ms_per_launch": kern_ms,
                         "kernel_share_of_step": r["kernel_ms"] / (avg_ms * args.steps),
                         "peak_source": pk["source"]},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "shots/s", "h2d_bytes_per_step": e2e["h2d_bytes_per_step"],
                    "d2h_bytes_per_step": e2e["d2h_bytes_per_step"]},
            "gpu_launches": r["launches"],
            "clocks": clocks,
            "extra_configs": extra,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
