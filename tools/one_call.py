"""One sample call of a config (for launch lists): python tools/one_call.py CFG SHOTS"""
import sys
sys.path.insert(0, '.')
import torch
from paper_2604_27058_b200.program import Program
from paper_2604_27058_b200.engine import DeviceProgram
cfg, shots = int(sys.argv[1]), int(sys.argv[2])
dp = DeviceProgram(Program.load(f'paper_2604_27058_b200/programs/c{cfg}.npz'))
out = dp.alloc_device_outputs(shots)
dp.sample_device(shots, out, seed=1)
torch.cuda.synchronize()
print("status", int(out['status'].item()))
