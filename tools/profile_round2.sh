#!/bin/bash
# Round-2 captures (GPU box, after the plain commands exit 0): one `ncu --set full` of each
# config's timed kernel, and the per-launch DRAM bytes + duration of every config-3 fused pass.
set -u
N="ncu --set full --clock-control none --import-source on"
M="ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv"
python tools/one_call.py 0 100000 >/dev/null && \
  $N -k regex:fs_jit_general -c 1 -o gpurun_out/r2_prof_c0_gjit python tools/one_call.py 0 100000 >/dev/null 2>&1
python tools/one_call.py 2 10000000 >/dev/null && \
  $N -k regex:fs_jit_general -c 1 -o gpurun_out/r2_prof_c2_gjit python tools/one_call.py 2 10000000 >/dev/null 2>&1
python tools/one_call.py 3 1000 >/dev/null && \
  $M -k regex:fs_pass --log-file gpurun_out/r2_c3_passes.csv python tools/one_call.py 3 1000 >/dev/null 2>&1
python tools/one_call.py 3 64 >/dev/null && \
  $N -k regex:fs_pass_42 -c 1 -o gpurun_out/r2_prof_c3_p42 python tools/one_call.py 3 64 >/dev/null 2>&1
bash tools/profile_c4.sh   # config 4: launch list + one capture per specialised segment form
ls -la gpurun_out/r2_prof_*.ncu-rep gpurun_out/r2_c3_passes.csv
