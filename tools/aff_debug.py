"""Compare the affine kernel with the other frame paths and the oracle on one golden program.
python tools/aff_debug.py NAME"""
import os, sys
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np
import oracle
from goldens import load
from paper_2604_27058_b200._abi import FS_RNG_PHILOX, FS_NO_JIT, FS_FORCE_GENERAL
from paper_2604_27058_b200.engine import DeviceProgram
name = sys.argv[1]
P = load(name)["prog"]
dp = DeviceProgram(P)
n = 2048
_, o, _ = oracle.sample(P, n, seed=77, shot0=64, flags=FS_RNG_PHILOX)
res = {}
for label, env, fl in (("affine", None, 0), ("faultlist", "FS_NO_AFFINE", 0), ("interp", None, FS_NO_JIT),
                       ("general", None, FS_FORCE_GENERAL)):
    if env: os.environ[env] = "1"
    _, g, _ = dp.sample_host(n, seed=77, shot0=64, flags=FS_RNG_PHILOX | fl)
    if env: del os.environ[env]
    res[label] = g
    for attr in ("meas", "det", "obs", "accepted"):
        a, b = np.asarray(getattr(g, attr)), np.asarray(getattr(o, attr))
        if not np.array_equal(a, b):
            d = np.argwhere(a != b)
            print(label, attr, "mismatch", len(d), "first", d[:6].tolist())
    print(label, "jit:", dp.jit_status())
print("meas rows", o.meas.shape, "det", o.det.shape)
