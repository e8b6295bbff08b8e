export NCCL_DEBUG=WARN
echo "== peer all-reduce latency: memory ordering variants (chain of 32 dependent all-reduces, graph replay)"
for n in 4 2; do for mb in 1 4 16; do for v in "SPX_PEER_ORDER=0" "SPX_PEER_ORDER=1" "SPX_PEER_ORDER=3" "SPX_PEER_ORDER=1 SPX_PEER_TWOSHOT=0"; do
  r=$(env $v timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29700 + n*10 + mb)) tools/peer_bench.py --mb $mb 2>/dev/null | grep "{" | tail -1)
  echo "n=$n mb=$mb [$v] $r"
done; done; done
echo "== off-critical-path peer grid cap (ZeRO-3 prefetch gathers, gradient reduce-scatters) at N=4"
for b in 0 16 32 64; do
  SPX_PEER_OFFCRIT_BLOCKS=$b timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29800 + b)) bench.py --gpus 4 --steps 8 --warmup 3 --config c3 --no-cpu-baseline --e2e-seconds 3 > gpurun_out/r2c_c3_ob$b.log 2>&1
  SPX_PEER_OFFCRIT_BLOCKS=$b timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29900 + b)) bench.py --gpus 4 --steps 30 --warmup 3 --config c5 --no-cpu-baseline --e2e-seconds 3 > gpurun_out/r2c_c5_ob$b.log 2>&1
done
python tools/bench_summary.py gpurun_out/r2c_*.log
echo "== dynamic GEMM unit scheduling off (SPX_H3_DYNAMIC=0) at N=4"
SPX_H3_DYNAMIC=0 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29990 bench.py --gpus 4 --steps 8 --warmup 3 --config c3 --no-cpu-baseline --e2e-seconds 3 > gpurun_out/r2c_c3_dyn0.log 2>&1
SPX_H3_DYNAMIC=0 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29991 bench.py --gpus 4 --steps 30 --warmup 3 --config c5 --no-cpu-baseline --e2e-seconds 3 > gpurun_out/r2c_c5_dyn0.log 2>&1
python tools/bench_summary.py gpurun_out/r2c_c3_dyn0.log gpurun_out/r2c_c5_dyn0.log
