"""Stratified sampling rate: python tools/stratum_speed.py CFG SHOTS W"""
import sys, time
sys.path.insert(0, '.')
import torch
from paper_2604_27058_b200.program import Program
from paper_2604_27058_b200.engine import DeviceProgram
cfg, n, w = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
dp = DeviceProgram(Program.load(f'paper_2604_27058_b200/programs/c{cfg}.npz'))
out = dp.alloc_device_outputs(n)
dp.sample_stratum_device(w, n, out, seed=1)
torch.cuda.synchronize()
for flags in (0, 1):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); dp.sample_stratum_device(w, n, out, seed=2, flags=flags); e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"config {cfg} w={w} {'splitmix' if flags else 'philox'}: {ms:.2f} ms / {n} shots = {n / ms * 1e3:.3e} shots/s, weight {dp.stratum_weight(w):.6e}")
