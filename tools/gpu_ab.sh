# A/B timing of variant builds: tools/gpu_ab.sh v1 v2 ... (default = the in-tree library)
cd $GRAFT_REPO_ROOT
for v in "$@"; do
  if [ $v = default ]; then L=""; else L="--lib paper_2408_10743_b200/_variants/$v/libsymdist_b200.so"; fi
  timeout 300 python tools/exp.py time $L --configs 4,5 --gmax 9 >> gpurun_out/ab.log 2>&1
done
cat gpurun_out/ab.log
