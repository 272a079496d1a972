# variants of the affine kernel on config 1 (GPU box)
for v in "FS_AFF_PARENTS=6" "FS_AFF_PARENTS=3" "FS_AFF_PARENTS=2" "FS_AFF_PARENTS=1" "FS_AFF_NO_DIFF=1"; do echo "$v"; env $v python tools/aff_check.py 1 | tail -1; done
