export NCCL_DEBUG=WARN
mkdir -p gpurun_out
for v in 0 16 32; do for c in c2 c5; do
  SPX_SIDE_GEMM_RESERVE=$v timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29604 bench.py --gpus 4 --steps 30 --warmup 5 --config $c --no-cpu-baseline > gpurun_out/r2t_${c}_r$v.log 2>&1
  echo "reserve=$v $(python tools/bench_summary.py gpurun_out/r2t_${c}_r$v.log | cut -c1-260)"
done; done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29605 bench.py --gpus 4 --steps 30 --warmup 5 --config c4 --no-cpu-baseline > gpurun_out/r2t_c4.log 2>&1
echo "c4 $(python tools/bench_summary.py gpurun_out/r2t_c4.log | cut -c1-260)"
