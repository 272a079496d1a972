#!/bin/bash
# GPU box: bench line, launch list of the bench command, one ncu --set full capture of the
# config-1 dominant kernel.  Outputs in gpurun_out/.
set -u
python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:fs_aff_frame -c 1 -o gpurun_out/prof_c1_aff \
  python tools/one_call.py 1 10000000 > gpurun_out/ncu_aff.log 2>&1
ls -la gpurun_out/*.ncu-rep gpurun_out/launches.csv
ncu --set full --clock-control none --import-source on -k regex:fs_jit_general -c 1 -o gpurun_out/prof_c2_gjit \
  python tools/one_call.py 2 10000000 > gpurun_out/ncu_c2.log 2>&1
