"""Write the affine frame kernel source a program would get (host generator, no GPU), and
optionally compile it offline to SASS:  python tools/aff_src.py CFG OUT.cu [--sass]"""
import ctypes as C
import subprocess
import sys

sys.path.insert(0, ".")
from paper_2604_27058_b200 import _lib  # noqa: E402
from paper_2604_27058_b200._abi import DescHolder  # noqa: E402
from paper_2604_27058_b200.program import Program  # noqa: E402

cfg, out = sys.argv[1], sys.argv[2]
P = Program.load(f"paper_2604_27058_b200/programs/c{cfg}.npz" if cfg.isdigit() else cfg)
L = _lib.lib()
h = DescHolder(P)
buf = C.create_string_buffer(1 << 24)
L.fs_debug_aff_source.argtypes = [C.c_void_p, C.c_char_p, C.c_size_t]
L.fs_debug_aff_source(C.byref(h.desc), buf, 1 << 24)
open(out, "w").write(buf.value.decode())
if "--sass" in sys.argv:
    cub = out.rsplit(".", 1)[0] + ".cubin"
    r = subprocess.run(["nvcc", "-cubin", "-arch=sm_100a", "-std=c++17", "-lineinfo", "-Ipaper_2604_27058_b200/csrc",
                        "-Iinclude", "-DFS_JIT=1", "-Xptxas", "-v", "-o", cub, out], capture_output=True, text=True)
    print(r.stderr[-600:])
