#!/bin/bash
# Iteration call: GPU tests, kernel timings (tools/t4.py), bench without the CPU leg.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/t4.py > gpurun_out/t4.log 2>&1
for v in paper_2408_10743_b200/_variants/*/; do
  [ -f $v/libsymdist_b200.so ] && SDB_LIBRARY=$v/libsymdist_b200.so timeout 300 python tools/t4.py >> gpurun_out/t4.log 2>&1
done
timeout 600 python bench.py --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
echo done
