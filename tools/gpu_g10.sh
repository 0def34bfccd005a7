cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_tile_kernel -s 4 -c 1 -o gpurun_out/g10_noprod python tools/exp.py time --lib paper_2408_10743_b200/_variants/noprod/libsymdist_b200.so --configs 4 --gmax 9 > gpurun_out/g10.log 2>&1
tail -2 gpurun_out/g10.log
