"""Generate the affine frame kernel of a config here (no GPU) and report ptxas registers/spills.
python tools/aff_regs.py CFG"""
import sys, ctypes as C, subprocess, os
sys.path.insert(0, '.')
from paper_2604_27058_b200 import _lib
from paper_2604_27058_b200._abi import DescHolder
from paper_2604_27058_b200.program import Program
cfg = sys.argv[1]
P = Program.load(cfg if cfg.endswith('.npz') else f'paper_2604_27058_b200/programs/c{cfg}.npz')
h = DescHolder(P)
L = _lib.lib()
L.fs_debug_aff_source.argtypes = [C.c_void_p, C.c_char_p, C.c_size_t]
n = L.fs_debug_aff_source(C.byref(h.desc), None, 0)
if n < 0:
    sys.exit(f'not applicable ({n})')
buf = C.create_string_buffer(n + 1)
L.fs_debug_aff_source(C.byref(h.desc), buf, n + 1)
path = f'/tmp/aff_c{os.path.basename(cfg)}.cu'
open(path, 'w').write(buf.value.decode())
inc = os.path.abspath('paper_2604_27058_b200/csrc')
r = subprocess.run(['nvcc', '-cubin', '-arch=sm_100a', '-O3', '-std=c++17', '-lineinfo', '-I', inc, '-I', 'include', '-Xptxas', '-v',
                    '-o', path.replace('.cu', '.cubin'), path], capture_output=True, text=True)
print('\n'.join(l for l in r.stderr.splitlines() if 'fs_aff' in l or 'registers' in l or 'spill' in l or 'error' in l))
print(path)
