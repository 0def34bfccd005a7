cd $GRAFT_REPO_ROOT
timeout 600 python tools/exp.py check --kernels 0 > gpurun_out/g11.log 2>&1
timeout 300 python tools/exp.py time --lib paper_2408_10743_b200/_variants/noprod/libsymdist_b200.so --configs 4,5 --gmax 9 >> gpurun_out/g11.log 2>&1
cat gpurun_out/g11.log
