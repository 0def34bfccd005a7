# Quick A/B on the GPU box: parity check of the tensor-core kernel on the reference goldens,
# level timings, optional microbenchmarks. Usage: tools/gpu_quick.sh [microbench binaries...]
cd $GRAFT_REPO_ROOT
timeout 900 python tools/exp.py check --kernels 0,4 --configs 1,2,4,5 > gpurun_out/quick_check.log 2>&1
for v in default $VARIANTS; do
  if [ $v = default ]; then L=""; else L="--lib paper_2408_10743_b200/_variants/$v/libsymdist_b200.so"; fi
  timeout 300 python tools/exp.py time $L --configs 4,5 --gmax 9 >> gpurun_out/quick_time.log 2>&1
done
for b in "$@"; do timeout 300 $b > gpurun_out/quick_$(basename $b).log 2>&1; done
cat gpurun_out/quick_check.log gpurun_out/quick_time.log
for b in "$@"; do cat gpurun_out/quick_$(basename $b).log; done
