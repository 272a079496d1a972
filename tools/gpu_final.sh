#!/bin/bash
# Round-end validation on one B200: build, smoke, the full GPU suite, the bench line.
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo rc=$? >> gpurun_out/final_smoke.log
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/final_gpu.log 2>&1; echo rc=$? >> gpurun_out/final_gpu.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo rc=$? >> gpurun_out/final_bench.err
