cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_tile_kernel -s 4 -c 1 -o gpurun_out/g15_tc python tools/exp.py time --configs 4 --gmax 9 > gpurun_out/g15.log 2>&1
tail -1 gpurun_out/g15.log
