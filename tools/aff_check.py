"""Affine frame kernel vs the fault-list frame kernel: bit-exact outputs + timing.
python tools/aff_check.py [CFG ...]"""
import os, sys, json
sys.path.insert(0, '.')
import torch
from paper_2604_27058_b200.program import Program
from paper_2604_27058_b200.engine import DeviceProgram
from paper_2604_27058_b200.configs import CONFIGS

def run(dps, shots, seed, aff):
    dp = dps[0] if aff else dps[1]  # FS_NO_AFFINE is read when a program handle is created
    out = dp.alloc_device_outputs(shots)
    dp.sample_device(shots, out, seed=seed); torch.cuda.synchronize()
    ms = []
    for s in range(5):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); dp.sample_device(shots, out, seed=seed); e1.record(); torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    return out, min(ms)

for cfg in [int(c) for c in sys.argv[1:]] or [1]:
    P = Program.load(f'paper_2604_27058_b200/programs/c{cfg}.npz')
    os.environ.pop('FS_NO_AFFINE', None)
    dp = DeviceProgram(P)
    os.environ['FS_NO_AFFINE'] = '1'
    dp2 = DeviceProgram(P)
    os.environ.pop('FS_NO_AFFINE', None)
    for shots in (1000, 100003, CONFIGS[cfg]['shots']):
        a, ta = run((dp, dp2), shots, 7, True)
        b, tb = run((dp, dp2), shots, 7, False)
        same = all(torch.equal(a[k], b[k]) for k in a if k != 'status' and a[k] is not None)
        print(json.dumps({"cfg": cfg, "shots": shots, "equal": same, "aff_ms": ta, "old_ms": tb,
                          "aff_shots_per_s": shots / ta * 1e3}), flush=True)
    dp.close()
