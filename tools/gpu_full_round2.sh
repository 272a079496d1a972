set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2_smoke.log 2>&1; echo rc=$? >> gpurun_out/r2_smoke.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2_gpufull.log 2>&1; echo rc=$? >> gpurun_out/r2_gpufull.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench3.json 2> gpurun_out/r2_bench3.err; echo rc=$? >> gpurun_out/r2_bench3.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_bench_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/r2_ncu_launches.log 2>&1
timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:fs_aff_frame -c 1 --csv --log-file gpurun_out/r2_traffic_c1.csv python tools/one_call.py 1 10000000 > /dev/null 2>&1
timeout 1200 bash tools/profile_round2.sh > gpurun_out/r2_profile_round2.log 2>&1
