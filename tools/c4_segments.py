"""Per-segment census of a post-selected config: [begin, end), k, shots in, kernel ms.
python tools/c4_segments.py CFG SHOTS"""
import sys, ctypes as C
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2604_27058_b200.program import Program
from paper_2604_27058_b200.engine import DeviceProgram
cfg, shots = int(sys.argv[1]), int(sys.argv[2])
P = Program.load(f'paper_2604_27058_b200/programs/c{cfg}.npz')
dp = DeviceProgram(P)
out = dp.alloc_device_outputs(shots)
dp.sample_device(shots, out, seed=1); torch.cuda.synchronize()
L = dp._lib
L.fs_debug_kernel_timer.argtypes = [C.c_void_p, C.c_int]
L.fs_debug_kernel_times.restype = C.c_int64
L.fs_debug_kernel_times.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.c_int64]
L.fs_debug_seg_counts.argtypes = [C.c_void_p, C.POINTER(C.c_uint32), C.c_int]
L.fs_debug_kernel_timer(dp._h, 1)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); dp.sample_device(shots, out, seed=2); e1.record(); torch.cuda.synchronize()
t = (C.c_double * 4096)(); n = L.fs_debug_kernel_times(dp._h, t, 4096)
cb = (C.c_uint32 * 4096)(); nc = L.fs_debug_seg_counts(dp._h, cb, 4096)
ops = P.instrs[:, 0] & 0xFF
sched = P.schedule if hasattr(P, 'schedule') else None
bounds = [0] + [int(i) + 1 for i in np.nonzero(ops == 14)[0] if i + 1 < P.num_instrs] + [P.num_instrs]
print("total ms", e0.elapsed_time(e1), "launches", n, "counts", list(cb[:nc])[:40])
sch = np.asarray(sched)
for si, (b, e) in enumerate(zip(bounds[:-1], bounds[1:])):
    kin = int(sch[b - 1]) if b > 0 else 0
    karr = max([kin] + [int(x) for x in sch[b:e]])
    opc = np.bincount(ops[b:e], minlength=20)
    print(f"seg {si:2d} [{b:4d},{e:4d}) karr={karr:2d} in={cb[si] if si < nc else '-':>9} ms={t[si] if si < n else float('nan'):8.3f} "
          f"frame={opc[0]} noise={opc[11]} arr={opc[1]+opc[2]+opc[4]+opc[7]+opc[8]+opc[9]} meas={opc[5]+opc[6]}")
