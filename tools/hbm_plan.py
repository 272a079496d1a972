import sys, ctypes as C
sys.path.insert(0, '.')
from paper_2604_27058_b200.program import Program
from paper_2604_27058_b200.engine import DeviceProgram
P = Program.load('paper_2604_27058_b200/programs/c3.npz')
dp = DeviceProgram(P)
out = (C.c_int64 * 9)()
dp._lib.fs_debug_hbm_plan.argtypes = [C.c_void_p, C.POINTER(C.c_int64)]
print(dp._lib.fs_debug_hbm_plan(dp._h, out), list(out), "(steps, passes, fused ops, unfused array kernels, measurements, smem exchanges, reg mixing ops, diag runs, code words)")
import numpy as np, collections
buf = np.zeros((5000, 5), np.int32)
dp._lib.fs_debug_hbm_tileops.restype = C.c_int64
n = dp._lib.fs_debug_hbm_tileops(dp._h, buf.ctypes.data_as(C.POINTER(C.c_int32)), 5000)
ops = buf[:n]
names = ['H', 'S', 'SDAG', 'CX', 'CZ', 'ROT', 'EXPAND']
c = collections.Counter()
for ps, k, la, lb, dr in ops:
    m = lb if k == 3 else la
    where = '' if k in (1, 2, 4, 5) else ('reg' if m >= 8 else 'thr')
    c[names[k] + where] += 1
print(n, dict(c))
runs = [dr for *_, dr in ops if dr > 0]
print('diag runs', len(runs), 'mean len', np.mean(runs), 'hist', np.bincount(runs)[:20])
m = collections.Counter()
for ps, k, la, lb, dr in ops:
    if k in (0, 3, 6):
        mm = lb if k == 3 else la
        if mm < 8:
            m[int(mm)] += 1
print('exchanges by thread bit', sorted(m.items()))
