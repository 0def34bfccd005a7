cd $GRAFT_REPO_ROOT
timeout 600 python tools/exp.py check --kernels 0,4 > gpurun_out/g19.log 2>&1
SDB_TRACE_HOST=1 timeout 300 python tools/exp.py time --configs 4,5 --gmax 9 2>&1 | grep -E "tensor-core|k0" >> gpurun_out/g19.log
for f in 9:5:5 9:5:8 9:5:10 9:5:11 9:5:12 9:6:10 9:4:10; do
  echo "force $f" >> gpurun_out/g19.log
  SDB_TC_FORCE=$f timeout 300 python tools/exp.py time --configs 4 --gmax 9 >> gpurun_out/g19.log 2>&1
done
cat gpurun_out/g19.log
