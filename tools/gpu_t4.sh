#!/bin/bash
# GPU tests, then tools/t4.py timing three times (default build and any _variants/).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
: > gpurun_out/t4.log
for rep in 1 2 3; do
  timeout 300 python tools/t4.py >> gpurun_out/t4.log 2>&1
  for v in paper_2408_10743_b200/_variants/*/; do
    [ -f $v/libsymdist_b200.so ] && SDB_LIBRARY=$v/libsymdist_b200.so timeout 300 python tools/t4.py >> gpurun_out/t4.log 2>&1
  done
done
echo done
