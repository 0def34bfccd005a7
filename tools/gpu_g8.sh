cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_tile_kernel -s 4 -c 1 -o gpurun_out/g8_tc_g9 python bench.py --steps 1 --warmup 1 --no-extras --no-cpu > gpurun_out/g8_ncu.log 2>&1
tail -2 gpurun_out/g8_ncu.log
