cd $GRAFT_REPO_ROOT
timeout 600 python tools/exp.py check --kernels 0 --configs 1,2,4,5 2>&1 | cut -c1-150
bash tools/gpu_g21.sh
