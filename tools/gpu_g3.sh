cd $GRAFT_REPO_ROOT
SDB_TRACE_HOST=1 timeout 300 python tools/exp.py time --lib paper_2408_10743_b200/_variants/tcprof/libsymdist_b200.so --configs 4,5 > gpurun_out/g3_prof.log 2>&1
tail -40 gpurun_out/g3_prof.log
