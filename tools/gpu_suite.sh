# The round-end evidence in one call: GPU tests (plain, and optionally the bounds-checked build
# with CHECKED=1), the bench line, the reference arm, the launch list and one ncu --set full of
# the g = 9 tensor-core launch.
cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/suite_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/suite_pytest.log
if [ -n "$CHECKED" ]; then
SDB_TEST_VARIANT=checked timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/suite_checked.log 2>&1; echo "rc=$?" >> gpurun_out/suite_checked.log
fi
timeout 1200 python bench.py > gpurun_out/suite_bench.log 2> gpurun_out/suite_bench.err; echo "bench rc=$?" >> gpurun_out/suite_bench.err
timeout 900 python bench.py --impl reference --steps 5 --warmup 2 > gpurun_out/suite_ref.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/suite_launches.csv python bench.py --steps 1 --warmup 1 --no-extras --no-cpu > gpurun_out/suite_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_tile_kernel -s 4 -c 1 -o gpurun_out/suite_tc_g9 python bench.py --steps 1 --warmup 1 --no-extras --no-cpu > gpurun_out/suite_ncu_full.log 2>&1
tail -2 gpurun_out/suite_pytest.log; tail -1 gpurun_out/suite_bench.err; cat gpurun_out/suite_bench.log
