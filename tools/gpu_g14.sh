cd $GRAFT_REPO_ROOT
bash tools/gpu_ab.sh default fa ut16 > /dev/null 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/g14_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/g14_pytest.log
cat gpurun_out/ab.log; tail -3 gpurun_out/g14_pytest.log
