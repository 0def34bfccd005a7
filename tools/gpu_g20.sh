cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/g20_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/g20_pytest.log
tail -3 gpurun_out/g20_pytest.log
