export NCCL_DEBUG=WARN
for b in 0 64 96 120; do
  SPX_PEER_OFFCRIT_BLOCKS=$b SPX_PEER_OFFCRIT_MIN_BYTES=16777216 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29800 + b)) bench.py --gpus 4 --steps 8 --warmup 3 --config c3 --no-cpu-baseline --e2e-seconds 3 > gpurun_out/r2i_c3_ob$b.log 2>&1
done
for b in 0 64 96; do
  SPX_PEER_OFFCRIT_BLOCKS=$b SPX_PEER_OFFCRIT_MIN_BYTES=16777216 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29900 + b)) bench.py --gpus 2 --steps 8 --warmup 3 --config c3 --no-cpu-baseline --e2e-seconds 3 > gpurun_out/r2i_c3n2_ob$b.log 2>&1
done
SPX_PEER_OFFCRIT_BLOCKS=96 SPX_PEER_OFFCRIT_MIN_BYTES=16777216 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29990 bench.py --gpus 4 --steps 30 --warmup 3 --config c5 --no-cpu-baseline --e2e-seconds 3 > gpurun_out/r2i_c5_ob96.log 2>&1
python tools/bench_summary.py gpurun_out/r2i_*.log
