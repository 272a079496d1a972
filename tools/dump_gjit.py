"""Write the specialised general kernel source of a config to gpurun_out/gjit_cN.cu (needs a GPU)."""
import sys, ctypes as C
sys.path.insert(0, '.')
from paper_2604_27058_b200.program import Program
from paper_2604_27058_b200.engine import DeviceProgram
cfg = int(sys.argv[1])
dp = DeviceProgram(Program.load(f'paper_2604_27058_b200/programs/c{cfg}.npz'))
L = dp._lib
L.fs_debug_gjit_source.argtypes = [C.c_void_p, C.c_char_p, C.c_size_t]
n = L.fs_debug_gjit_source(dp._h, None, 0)
buf = C.create_string_buffer(n + 1)
L.fs_debug_gjit_source(dp._h, buf, n + 1)
open(f'gpurun_out/gjit_c{cfg}.cu', 'w').write(buf.value.decode())
print(n)
