"""End-to-end formatted output rate: python tools/fmt_speed.py CFG SHOTS FORMAT"""
import sys, time, io
sys.path.insert(0, '.')
import torch
from paper_2604_27058_b200.program import Program
from paper_2604_27058_b200 import runtime
cfg, shots, fmt = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
P = Program.load(f'paper_2604_27058_b200/programs/c{cfg}.npz')


class Sink:
    n = 0

    def write(self, b):
        self.n += len(b)


runtime.write_samples(P, 1 << 20, Sink(), format=fmt, rng="philox")
torch.cuda.synchronize()
for chunk in (1 << 20, 1 << 22):
    s = Sink()
    t0 = time.perf_counter()
    runtime.write_samples(P, shots, s, format=fmt, rng="philox", chunk=chunk)
    dt = time.perf_counter() - t0
    print(f"config {cfg} {fmt} chunk={chunk}: {shots / dt:.3e} shots/s, {s.n / dt / 1e9:.2f} GB/s out, {s.n} bytes")
