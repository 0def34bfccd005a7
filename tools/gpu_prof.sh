#!/bin/bash
# ncu --set full of one tensor-core tile launch (default: config 4's g = 9 launch, the 5th
# tc_tile_kernel launch of a bench step with one warm-up step), after a plain run of the same
# command. Usage: tools/gpu_prof.sh <tag> [skip] [config]
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${1:-prof}; SKIP=${2:-4}; CFG=${3:-4}
CMD="python bench.py --steps 1 --warmup 1 --no-extras --no-cpu --config $CFG"
$CMD > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_tile_kernel -s $SKIP -c 1 \
  -o gpurun_out/$TAG $CMD > gpurun_out/ncu_$TAG.log 2>&1
echo "rc=$?"
