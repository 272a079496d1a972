# time the affine kernel of config 1 at several warps-per-block settings (GPU box)
for wps in ${@:-12 16 20 24}; do echo "warps=$wps"; FS_AFF_WARPS=$wps python tools/aff_check.py 1 | tail -1; done
