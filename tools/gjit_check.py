"""General JIT vs general interpreter (bit-exact outputs) + timing: python tools/gjit_check.py CFG [shots]"""
import os, sys, json
sys.path.insert(0, '.')
import torch
from paper_2604_27058_b200.program import Program
from paper_2604_27058_b200.engine import DeviceProgram
from paper_2604_27058_b200._abi import FS_NO_JIT
from paper_2604_27058_b200.configs import CONFIGS
cfg = int(sys.argv[1]); shots = int(sys.argv[2]) if len(sys.argv) > 2 else CONFIGS[cfg]['shots']
P = Program.load(f'paper_2604_27058_b200/programs/c{cfg}.npz')
dp = DeviceProgram(P)
def run(flags):
    out = dp.alloc_device_outputs(shots)
    dp.sample_device(shots, out, seed=3, flags=flags); torch.cuda.synchronize()
    ms = []
    for s in range(3):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); dp.sample_device(shots, out, seed=3, flags=flags); e1.record(); torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    return out, min(ms)
a, ta = run(0)
b, tb = run(FS_NO_JIT)
same = all(torch.equal(a[k], b[k]) for k in a if k != 'status')
print(json.dumps({"cfg": cfg, "shots": shots, "equal": same, "jit_ms": ta, "interp_ms": tb, "jit": dp.jit_status()}))
