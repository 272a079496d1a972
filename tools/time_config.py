"""Time one config on the GPU: python tools/time_config.py CFG [shots] [steps]"""
import sys, time, json
sys.path.insert(0, '.')
import torch
from paper_2604_27058_b200.program import Program
from paper_2604_27058_b200.engine import DeviceProgram
cfg = int(sys.argv[1]); shots = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2] else None; steps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
from paper_2604_27058_b200.configs import CONFIGS
shots = shots or CONFIGS[cfg]['shots']
P = Program.load(f'paper_2604_27058_b200/programs/c{cfg}.npz')
dp = DeviceProgram(P)
out = dp.alloc_device_outputs(shots)
dp.sample_device(min(shots, 64), out, seed=1); torch.cuda.synchronize()
res = []
for s in range(steps):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); dp.sample_device(shots, out, seed=s); e1.record(); torch.cuda.synchronize()
    res.append(e0.elapsed_time(e1))
print(json.dumps({"config": cfg, "engine": dp.engine(0), "shots": shots, "ms": res, "shots_per_s": shots / (min(res) / 1e3), "status": int(out['status'].item())}))
