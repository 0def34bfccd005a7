cd $GRAFT_REPO_ROOT
timeout 600 tools/microbench/tc_pipe 6000 > gpurun_out/g4_tc_pipe.log 2>&1
cat gpurun_out/g4_tc_pipe.log
