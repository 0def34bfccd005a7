cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/g2_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/g2_pytest.log
timeout 900 python bench.py > gpurun_out/g2_bench.log 2> gpurun_out/g2_bench.err; echo "bench rc=$?" >> gpurun_out/g2_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/g2_launches.csv python bench.py --steps 1 --warmup 1 --no-extras --no-cpu > gpurun_out/g2_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_tile_kernel -s 4 -c 1 -o gpurun_out/g2_tc_g9 python bench.py --steps 1 --warmup 1 --no-extras --no-cpu > gpurun_out/g2_ncu_full.log 2>&1
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_cases.py > gpurun_out/g2_memcheck.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/g2_memcheck.log
tail -3 gpurun_out/g2_pytest.log
