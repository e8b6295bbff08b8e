export NCCL_DEBUG=WARN
mkdir -p gpurun_out
for v in 1 0; do
  SPX_PREFETCH_SPLITS=$v timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29604 bench.py --gpus 4 --steps 10 --warmup 5 --config c3 --no-cpu-baseline > gpurun_out/r2v_c3_p$v.log 2>&1
  echo "prefetch_splits=$v $(python tools/bench_summary.py gpurun_out/r2v_c3_p$v.log | cut -c1-300)"
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29514 tools/nccl_parity.py > gpurun_out/r2v_par_n4.log 2>&1
echo "parity N=4 rc=$?"; grep -v "^\[\|OMP_NUM\|^\*\*\*\|^NCCL version\|^\s*$" gpurun_out/r2v_par_n4.log | tail -1
