#!/bin/bash
# One `ncu --set full` capture of each engine's dominant kernel (run on the GPU box after the
# plain commands have exited 0).  Reports land in gpurun_out/prof_*.ncu-rep.
set -u
N="ncu --set full --clock-control none --import-source on"
python tools/one_call.py 1 10000000 >/dev/null && \
  $N -k regex:fs_jit_frame -c 1 -o gpurun_out/prof_c1_frame python tools/one_call.py 1 10000000 >/dev/null 2>&1
$N -k regex:fault_list -c 1 -o gpurun_out/prof_c1_flist python tools/one_call.py 1 10000000 >/dev/null 2>&1
python tools/one_call.py 2 10000000 >/dev/null && \
  $N -k regex:fs_jit_general -c 1 -o gpurun_out/prof_c2_gjit python tools/one_call.py 2 10000000 >/dev/null 2>&1
python tools/one_call.py 3 64 >/dev/null && \
  $N -k regex:hbm_fused_pass --launch-skip 3 -c 1 -o gpurun_out/prof_c3_pass python tools/one_call.py 3 64 >/dev/null 2>&1
python tools/one_call.py 4 4000000 >/dev/null && \
  $N -k regex:block_kernel -c 1 -o gpurun_out/prof_c4_block python tools/one_call.py 4 4000000 >/dev/null 2>&1
ls -la gpurun_out/prof_*.ncu-rep
