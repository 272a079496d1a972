"""Affine vs fault-list frame kernel on a golden frame-only program: python tools/aff_golden_time.py NAME [shots]"""
import os, sys, json
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import torch
from goldens import load
from paper_2604_27058_b200.engine import DeviceProgram
name = sys.argv[1]; shots = int(sys.argv[2]) if len(sys.argv) > 2 else 10_000_000
P = load(name)["prog"]
dp = DeviceProgram(P)
def run(aff):
    if aff: os.environ.pop('FS_NO_AFFINE', None)
    else: os.environ['FS_NO_AFFINE'] = '1'
    out = dp.alloc_device_outputs(shots)
    dp.sample_device(shots, out, seed=3); torch.cuda.synchronize()
    ms = []
    for s in range(3):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); dp.sample_device(shots, out, seed=3); e1.record(); torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    return out, min(ms)
a, ta = run(True)
b, tb = run(False)
same = all(torch.equal(a[k], b[k]) for k in a if k != 'status')
bits = P.output_bits()
print(json.dumps({"name": name, "shots": shots, "equal": same, "aff_ms": ta, "faultlist_ms": tb,
                  "out_bits_per_shot": bits, "aff_GBps": shots * bits / 8 / ta / 1e6, "jit": dp.jit_status()}))
