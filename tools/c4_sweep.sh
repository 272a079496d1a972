# config 4 engine knobs (GPU box): time 4M shots
for v in "X=0" "FS_BLOCK_K=8" "FS_BLOCK_K=10" "FS_BLOCK_K=11" "FS_BLOCK_JIT_WARP=1" "FS_BLOCK_NO_JIT=1"; do
  echo "$v"; env $v python tools/time_config.py 4 4000000 3 | tail -1; done
