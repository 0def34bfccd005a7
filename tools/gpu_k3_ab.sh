#!/bin/bash
# GPU tests, then package routes (config 4 Saved_1/2_Gamma) and config 5 (g <= 9) timings for the
# default build and each _variants/ build, twice.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
: > gpurun_out/k3ab.log
for rep in 1 2; do
  for v in default paper_2408_10743_b200/_variants/*/; do
    if [ "$v" = default ]; then unset SDB_LIBRARY; else export SDB_LIBRARY=$v/libsymdist_b200.so; fi
    echo "== $v" >> gpurun_out/k3ab.log
    timeout 300 python tools/t_pkg.py 2>&1 | grep "^4 " >> gpurun_out/k3ab.log
    timeout 300 python tools/t4.py 0 5 >> gpurun_out/k3ab.log 2>&1
  done
done
unset SDB_LIBRARY
echo done
