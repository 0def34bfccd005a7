# quick GPU check: traces vs goldens and timings for the default and forced tensor-core kernels
cd $GRAFT_REPO_ROOT
timeout 600 python tools/exp.py check --kernels 0,4 > gpurun_out/q_check.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "config4 or config5 or small_configs or oracle_agreement" >> gpurun_out/q_check.log 2>&1
cat gpurun_out/q_check.log | tail -20
