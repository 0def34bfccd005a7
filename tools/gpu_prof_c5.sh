cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/t4.py 0 5 > gpurun_out/t4_c5.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tile_kernel -s 5 -c 1 -o gpurun_out/prof_c5_g9 python tools/t4.py 0 5 > gpurun_out/ncu_c5.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_c5.log
