export NCCL_DEBUG=WARN
mkdir -p gpurun_out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29514 tools/nccl_parity.py > gpurun_out/r2o_par_n4.log 2>&1
echo "parity N=4 rc=$?"; grep -v "^\[\|OMP_NUM\|^\*\*\*\|^NCCL version\|^\s*$" gpurun_out/r2o_par_n4.log | tail -1
for N in 4 2; do for c in c3 c5 c2 c4; do
  [ $N = 2 ] && [ $c != c3 ] && [ $c != c5 ] && continue
  st=30; [ "$c" = c3 ] && st=10
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29600 + N)) bench.py --gpus $N --steps $st --warmup 5 --config $c --no-cpu-baseline > gpurun_out/r2o_${c}_n$N.log 2>&1
  python tools/bench_summary.py gpurun_out/r2o_${c}_n$N.log | cut -c1-300
done; done
