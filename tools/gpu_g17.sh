cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q -s -k "early_exit" > gpurun_out/g17_early.log 2>&1; echo "rc=$?" >> gpurun_out/g17_early.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/g17_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/g17_pytest.log
SDB_TEST_VARIANT=checked timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/g17_checked.log 2>&1; echo "rc=$?" >> gpurun_out/g17_checked.log
tail -3 gpurun_out/g17_early.log gpurun_out/g17_pytest.log gpurun_out/g17_checked.log; grep "skipped over" gpurun_out/g17_early.log
