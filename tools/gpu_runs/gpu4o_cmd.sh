export NCCL_DEBUG=WARN
mkdir -p gpurun_out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29514 tools/nccl_parity.py > gpurun_out/r2q_par_n4.log 2>&1
echo "parity N=4 rc=$?"; grep -v "^\[\|OMP_NUM\|^\*\*\*\|^NCCL version\|^\s*$" gpurun_out/r2q_par_n4.log | tail -1
for v in 8 0; do for c in c2 c5 c3; do
  st=30; [ "$c" = c3 ] && st=10
  SPX_HOIST_YIELD=$v timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29604 bench.py --gpus 4 --steps $st --warmup 5 --config $c --no-cpu-baseline > gpurun_out/r2q_${c}_y$v.log 2>&1
  echo "yield=$v $(python tools/bench_summary.py gpurun_out/r2q_${c}_y$v.log | cut -c1-300)"
done; done
