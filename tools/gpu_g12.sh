cd $GRAFT_REPO_ROOT
for f in 9:5:1 9:5:2 9:5:3 9:5:4 9:5:5 9:4:5 9:6:5 9:3:5; do
  echo "force $f" >> gpurun_out/g12.log
  SDB_TC_FORCE=$f timeout 300 python tools/exp.py time --configs 4 --gmax 9 >> gpurun_out/g12.log 2>&1
done
cat gpurun_out/g12.log
