for v in "FS_AFF_DIAG=0" "FS_AFF_ATOMIC_TERMS=1" "FS_AFF_DIAG=6" "FS_AFF_DIAG=0"; do echo "$v"; env $v python tools/aff_check.py 1 | tail -1; done
