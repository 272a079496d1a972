for v in "FS_GJIT_MB=4" "FS_GJIT_MB=5" "FS_GJIT_MB=6" "FS_GJIT_MB=8"; do echo "$v"; env $v python tools/gjit_check.py 2 | tail -1; done
