for v in "FS_GJIT_NREG=32" "FS_GJIT_NREG=40" "FS_GJIT_NREG=48" "FS_GJIT_NREG=24" "FS_GJIT_NREG=32"; do echo "$v"; env $v python tools/gjit_check.py 0 | tail -1; done
