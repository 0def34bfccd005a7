#!/bin/bash
# BASELINE config 5 to completion on one GPU, with nvidia-smi clocks/power sampled every 5 s.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=timestamp,clocks.sm,clocks.max.sm,power.draw,temperature.gpu,clocks_event_reasons.active \
  --format=csv -l 5 > gpurun_out/c5_clocks.csv 2>&1 &
SMI=$!
timeout 2400 python tools/config5_full.py > gpurun_out/config5_full.json 2> gpurun_out/config5_full.err
echo "rc=$?" >> gpurun_out/config5_full.err
kill $SMI
