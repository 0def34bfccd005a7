#!/bin/bash
# ncu --set full of one tile-kernel launch (config 4, level g=9: the 6th tile launch, g = 4..9).
# Usage: tools/gpu_prof.sh <tag> [skip] [config]
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${1:-prof}; SKIP=${2:-5}; CFG=${3:-4}
CMD="python bench.py --steps 1 --warmup 1 --no-extras --no-cpu --config $CFG"
$CMD > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tile_kernel -s $SKIP -c 1 \
  -o gpurun_out/$TAG $CMD > gpurun_out/ncu_$TAG.log 2>&1
echo "rc=$?"
