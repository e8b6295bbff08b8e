#!/bin/bash
# multi-GPU bench sweep on one box: tools/scale_runs.sh "2 4" "c2 c5 c4 c3" [tag]
NS=${1:-"2 4"}; CS=${2:-"c2"}; TAG=${3:-r}
export NCCL_DEBUG=WARN
for n in $NS; do for c in $CS; do
  st=30; [ "$c" = c3 ] && st=8
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $((29500 + n)) bench.py --gpus $n --steps $st --warmup 3 --config $c --no-cpu-baseline \
    > gpurun_out/${TAG}_${c}_n$n.log 2>&1
done; done
python tools/bench_summary.py gpurun_out/${TAG}_*.log
