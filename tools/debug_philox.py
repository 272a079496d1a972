import sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import oracle
from goldens import load
from paper_2604_27058_b200.engine import DeviceProgram
from paper_2604_27058_b200._abi import FS_FORCE_GENERAL
for name in ["config1", "toy_repetition", "toy_certain", "rand01"]:
    P = load(name)["prog"]
    dp = DeviceProgram(P)
    for shot0 in (0, 64):
        _, f, _ = dp.sample_host(2048, seed=77, shot0=shot0, flags=0)
        _, g, _ = dp.sample_host(2048, seed=77, shot0=shot0, flags=FS_FORCE_GENERAL)
        _, o, _ = oracle.sample(P, 2048, seed=77, shot0=shot0, flags=0)
        fm, gm, om = f.measurements(), g.measurements(), o.measurements()
        print(name, shot0, 'frame!=oracle', (fm != om).mean(), 'gen!=oracle', (gm != om).mean(), 'frame!=gen', (fm != gm).mean())
        if (fm != om).any():
            bad = np.nonzero((fm != om).any(0))[0]
            print('   first bad record cols', bad[:10], 'shots', np.nonzero((fm != om).any(1))[0][:10])
