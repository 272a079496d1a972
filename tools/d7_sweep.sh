for v in "FS_AFF_PAIRS=8" "FS_AFF_PAIRS=6" "FS_AFF_PAIRS=4" "FS_AFF_PAIRS=2"; do echo "$v"; env $v python tools/aff_golden_time.py aff_surface_d7 | tail -1; done
