#!/bin/bash
# Config-4 captures of the specialised segmented engine (GPU box, after the plain command exits 0):
# the launch list of one 2^23-shot chunk and one `ncu --set full` per segment form (lane / warp /
# CTA per shot).
set -u
N="ncu --set full --clock-control none --import-source on"
python tools/one_call.py 4 8388608 > /dev/null || exit 1
ncu --metrics gpu__time_duration.sum,sm__inst_executed.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none -c 60 --csv --log-file gpurun_out/r2h_c4_launches.csv python tools/one_call.py 4 8388608 > /dev/null 2>&1
$N -k fs_seg_50 -c 1 -f -o gpurun_out/r2h_c4_lane_seg50 python tools/one_call.py 4 8388608 > /dev/null 2>&1
$N -k fs_seg_75 -c 1 -f -o gpurun_out/r2h_c4_warp_seg75 python tools/one_call.py 4 8388608 > /dev/null 2>&1
$N -k fs_seg_276 -c 1 -f -o gpurun_out/r2h_c4_cta_seg276 python tools/one_call.py 4 8388608 > /dev/null 2>&1
ls -la gpurun_out/r2h_*
