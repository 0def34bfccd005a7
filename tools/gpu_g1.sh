cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/g1_smi.txt
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/g1_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/g1_pytest.log
timeout 600 python tools/exp.py check --kernels 0,4,2 > gpurun_out/g1_check.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/g1_bench.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/g1_launches.csv python bench.py --steps 1 --warmup 1 --no-extras --no-cpu > gpurun_out/g1_ncu.log 2>&1
tail -3 gpurun_out/g1_pytest.log
