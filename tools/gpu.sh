#!/bin/bash
# build the sm_100a library in-tree, then run a command on the GPU box
set -e
cd /root/repo
python paper_2401_11202_b200/build.py > /dev/null
T=${GPU_TIMEOUT:-900}
exec timeout $((T + 1700)) /usr/local/graft/bin/gpurun --timeout $T -- "$@"
