cd $GRAFT_REPO_ROOT
for v in default noprod nomma; do
  if [ $v = default ]; then L=""; else L="--lib paper_2408_10743_b200/_variants/$v/libsymdist_b200.so"; fi
  timeout 300 python tools/exp.py time $L --configs 4,5 --gmax 9 >> gpurun_out/g5.log 2>&1
done
SDB_TRACE_HOST=1 timeout 300 python tools/exp.py time --lib paper_2408_10743_b200/_variants/tcprof/libsymdist_b200.so --configs 4 --gmax 9 > gpurun_out/g5_prof.log 2>&1
cat gpurun_out/g5.log; grep -A3 "level 9" gpurun_out/g5_prof.log | tail -8
