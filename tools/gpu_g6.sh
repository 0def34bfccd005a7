cd $GRAFT_REPO_ROOT
for v in tcprof tcprof_noprod; do
SDB_TRACE_HOST=1 timeout 300 python tools/exp.py time --lib paper_2408_10743_b200/_variants/$v/libsymdist_b200.so --configs 4 --gmax 9 > gpurun_out/g6_$v.log 2>&1
echo $v; grep "stages 1[0-9][0-9][0-9][0-9]" gpurun_out/g6_$v.log | tail -1; grep -B1 -A1 "stages 1[0-9][0-9][0-9][0-9]" gpurun_out/g6_$v.log | grep epi | tail -2
done
