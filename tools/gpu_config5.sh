# config 5 ([[80,10]] seed 4) to its distance on one B200 (~10 min)
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw --format=csv -lms 5000 > gpurun_out/c5_smi.csv 2>&1 &
SMI=$!
SDB_TRACE_HOST=1 timeout 3000 python tools/exp.py config5 --gmax 0 > gpurun_out/c5_full.json 2> gpurun_out/c5_full.err
echo "rc=$?" >> gpurun_out/c5_full.err
kill $SMI
cat gpurun_out/c5_full.json; tail -3 gpurun_out/c5_full.err
