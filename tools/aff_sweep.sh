# time the affine kernel of config 1 at several warp-pair counts per block (GPU box)
for np in ${@:-8 10 12}; do echo "pairs=$np"; FS_AFF_PAIRS=$np python tools/aff_check.py 1 | tail -1; done
