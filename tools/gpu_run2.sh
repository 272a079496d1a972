set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_pins.py -q -m gpu > gpurun_out/r2_pins2.log 2>&1; echo rc=$? >> gpurun_out/r2_pins2.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r2_bench2.json 2> gpurun_out/r2_bench2.err; echo rc=$? >> gpurun_out/r2_bench2.err
python tools/one_call.py 1 10000000 > /dev/null && timeout 600 ncu --set full --clock-control none --import-source on -k regex:fs_aff_frame -c 1 -o gpurun_out/r2_prof_c1_aff python tools/one_call.py 1 10000000 > gpurun_out/r2_ncu_c1.log 2>&1
timeout 600 compute-sanitizer --tool racecheck --racecheck-report all python tools/one_call.py 1 100000 > gpurun_out/r2_racecheck_aff.log 2>&1; echo rc=$? >> gpurun_out/r2_racecheck_aff.log
timeout 600 compute-sanitizer --tool synccheck python tools/one_call.py 1 100000 > gpurun_out/r2_synccheck_aff.log 2>&1; echo rc=$? >> gpurun_out/r2_synccheck_aff.log
timeout 900 compute-sanitizer --tool racecheck --racecheck-report all python tools/one_call.py 3 2 > gpurun_out/r2_racecheck_pass.log 2>&1; echo rc=$? >> gpurun_out/r2_racecheck_pass.log
timeout 900 compute-sanitizer --tool synccheck python tools/one_call.py 3 2 > gpurun_out/r2_synccheck_pass.log 2>&1; echo rc=$? >> gpurun_out/r2_synccheck_pass.log
