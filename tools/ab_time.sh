# A/B: time config $1 ($2 shots) with the current library and with _ab/libfs_before.so
python tools/time_config.py $1 $2 3 | tail -1
cp paper_2604_27058_b200/_build/libfs_sampler.so _ab/libfs_new.so
cp _ab/libfs_before.so paper_2604_27058_b200/_build/libfs_sampler.so
python tools/time_config.py $1 $2 3 | tail -1
cp _ab/libfs_new.so paper_2604_27058_b200/_build/libfs_sampler.so
