cd $GRAFT_REPO_ROOT
timeout 600 python tools/exp.py check --kernels 0 > gpurun_out/g7.log 2>&1
timeout 300 python tools/exp.py time --lib paper_2408_10743_b200/_variants/noprod/libsymdist_b200.so --configs 4,5 --gmax 9 >> gpurun_out/g7.log 2>&1
SDB_TRACE_HOST=1 timeout 300 python tools/exp.py time --lib paper_2408_10743_b200/_variants/tcprof/libsymdist_b200.so --configs 4 --gmax 9 > gpurun_out/g7_prof.log 2>&1
cat gpurun_out/g7.log; grep "stages 1[0-9][0-9][0-9][0-9]" gpurun_out/g7_prof.log | tail -1; grep -B1 -A1 "stages 1[0-9][0-9][0-9][0-9]" gpurun_out/g7_prof.log | grep epi | tail -2
