cd $GRAFT_REPO_ROOT
timeout 120 tools/microbench/tc_pair 6000 > gpurun_out/g16_pair.log 2>&1; echo "rc=$?" >> gpurun_out/g16_pair.log
cat gpurun_out/g16_pair.log
