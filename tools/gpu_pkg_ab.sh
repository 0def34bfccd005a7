#!/bin/bash
# Package-route GPU tests, then tools/t_pkg.py three times for the default build and each _variants/ build.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
: > gpurun_out/t_pkg.log
for rep in 1 2 3; do
  echo "== default" >> gpurun_out/t_pkg.log; timeout 300 python tools/t_pkg.py >> gpurun_out/t_pkg.log 2>&1
  for v in paper_2408_10743_b200/_variants/*/; do
    echo "== $v" >> gpurun_out/t_pkg.log
    [ -f $v/libsymdist_b200.so ] && SDB_LIBRARY=$v/libsymdist_b200.so timeout 300 python tools/t_pkg.py >> gpurun_out/t_pkg.log 2>&1
  done
done
echo done
