export NCCL_DEBUG=WARN
mkdir -p gpurun_out
for N in 4 2; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29510+N)) tools/nccl_parity.py > gpurun_out/r2l_par_n$N.log 2>&1
  echo "parity N=$N rc=$?"; grep -v "^\[\|OMP_NUM\|^\*\*\*\|^NCCL version\|^\s*$" gpurun_out/r2l_par_n$N.log | tail -1
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29531 \
  tools/timeline.py --config c3 --json gpurun_out/r2l_tl_c3_n4.json > gpurun_out/r2l_tl_c3_n4.log 2> gpurun_out/r2l_tl_c3_n4.err
echo "timeline rc=$?"; head -1 gpurun_out/r2l_tl_c3_n4.log | cut -c1-600
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29532 \
  tools/timeline.py --config c2 --json gpurun_out/r2l_tl_c2_n4.json > gpurun_out/r2l_tl_c2_n4.log 2> gpurun_out/r2l_tl_c2_n4.err
head -1 gpurun_out/r2l_tl_c2_n4.log | cut -c1-600
for N in 4 2; do for c in c3 c2 c5 c4; do
  st=30; [ "$c" = c3 ] && st=10
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29600 + N)) bench.py --gpus $N --steps $st --warmup 5 --config $c --no-cpu-baseline > gpurun_out/r2l_${c}_n$N.log 2>&1
  python tools/bench_summary.py gpurun_out/r2l_${c}_n$N.log
done; done
