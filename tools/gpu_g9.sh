cd $GRAFT_REPO_ROOT
for v in noprod nomma; do
timeout 300 python tools/exp.py time --lib paper_2408_10743_b200/_variants/$v/libsymdist_b200.so --configs 4,5 --gmax 9 >> gpurun_out/g9.log 2>&1
done
cat gpurun_out/g9.log
