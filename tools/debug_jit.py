import sys, os, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import oracle
from goldens import load
from paper_2604_27058_b200.engine import DeviceProgram
from paper_2604_27058_b200._abi import FS_NO_JIT
for name in ["toy_repetition", "toy_certain", "config1"]:
    P = load(name)["prog"]
    dp = DeviceProgram(P)
    for n in (64, 4096):
        _, a, _ = dp.sample_host(n, seed=3, flags=0)
        _, b, _ = dp.sample_host(n, seed=3, flags=FS_NO_JIT)
        am, bm = a.measurements(), b.measurements()
        bad = np.nonzero((am != bm).any(1))[0]
        print(name, n, os.environ.get("FS_JIT_FLIPCAP"), 'mismatch shots', len(bad), bad[:8], dp.jit_status())
