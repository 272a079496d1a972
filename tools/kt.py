"""Per-kernel device time of one config via the library's kernel timer + total step time.
python tools/kt.py CFG SHOTS STEPS"""
import sys, json, ctypes as C
sys.path.insert(0, '.')
import torch
from paper_2604_27058_b200.program import Program
from paper_2604_27058_b200.engine import DeviceProgram
cfg, shots, steps = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
dp = DeviceProgram(Program.load(f'paper_2604_27058_b200/programs/c{cfg}.npz'))
out = dp.alloc_device_outputs(shots)
for _ in range(2): dp.sample_device(shots, out, seed=1)
torch.cuda.synchronize()
L = dp._lib
L.fs_debug_kernel_timer.argtypes = [C.c_void_p, C.c_int]
L.fs_debug_kernel_time.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_int64)]
L.fs_debug_kernel_timer(dp._h, 1)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for s in range(steps): dp.sample_device(shots, out, seed=s)
e1.record(); torch.cuda.synchronize()
kms, kn = C.c_double(), C.c_int64()
L.fs_debug_kernel_time(dp._h, C.byref(kms), C.byref(kn))
tot = e0.elapsed_time(e1)
print(json.dumps({"config": cfg, "step_ms": tot / steps, "kernel_ms": kms.value / steps, "other_ms": (tot - kms.value) / steps,
                  "shots_per_s": shots * steps / tot * 1e3, "status": int(out['status'].item())}))
