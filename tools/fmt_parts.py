"""Time the pieces of the formatted-output path for config CFG: sample, format, D2H, host copy."""
import sys, time
sys.path.insert(0, '.')
import torch
from paper_2604_27058_b200.program import Program
from paper_2604_27058_b200.engine import DeviceProgram
from paper_2604_27058_b200._abi import FS_FMT_BIN, FS_FMT_01
cfg, n = int(sys.argv[1]), int(sys.argv[2])
dp = DeviceProgram(Program.load(f'paper_2604_27058_b200/programs/c{cfg}.npz'))
w = dp.alloc_device_outputs(n)
for fmt in (FS_FMT_BIN, FS_FMT_01):
    cap = dp.format_bound(n, fmt, 0, "1")
    dev = torch.empty(cap, dtype=torch.uint8, device="cuda")
    t0 = time.perf_counter(); host = torch.empty(cap, dtype=torch.uint8, pin_memory=True); tp = time.perf_counter() - t0
    for rep in range(2):
        torch.cuda.synchronize()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        t0 = time.perf_counter()
        e[0].record(); dp.sample_device(n, w, seed=rep); e[1].record()
        nb, nk = dp.format_device(n, w, fmt, True, 0, "1", dev); e[2].record()
        host[:nb].copy_(dev[:nb], non_blocking=True); e[3].record(); torch.cuda.synchronize()
        t1 = time.perf_counter()
        b = host[:nb].numpy().tobytes()
        t2 = time.perf_counter()
    print(f"fmt={fmt} n={n} sample {e[0].elapsed_time(e[1]):.2f} ms, format {e[1].elapsed_time(e[2]):.2f} ms, "
          f"d2h {e[2].elapsed_time(e[3]):.2f} ms ({nb / e[2].elapsed_time(e[3]) / 1e6:.1f} GB/s), "
          f"tobytes {1e3 * (t2 - t1):.1f} ms, pin alloc {1e3 * tp:.1f} ms, bytes {nb}")
