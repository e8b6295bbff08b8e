#!/bin/bash
# build the sm_100a library in-tree, then run ONE shell command string on the GPU box
#   GPU_TIMEOUT=secs GPUS=n tools/gpu.sh '<command>'
set -e
cd /root/repo
python paper_2401_11202_b200/build.py > /dev/null
T=${GPU_TIMEOUT:-900}
exec timeout $((T + 1700)) /usr/local/graft/bin/gpurun --gpus ${GPUS:-1} --timeout $T -- "$1"
