export NCCL_DEBUG=WARN
for N in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29510+N)) tools/nccl_parity.py > gpurun_out/r2j_par_n$N.log 2>&1
  echo "parity N=$N rc=$?"; grep -v "^\[\|OMP_NUM\|^\*\*\*\|^NCCL version\|^\s*$" gpurun_out/r2j_par_n$N.log | tail -1
done
for N in 2 4; do for c in c3 c2 c4 c5; do
  st=30; [ "$c" = c3 ] && st=10
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29600 + N)) bench.py --gpus $N --steps $st --warmup 5 --config $c --no-cpu-baseline > gpurun_out/r2j_${c}_n$N.log 2>&1
done; done
python tools/bench_summary.py gpurun_out/r2j_c*.log
pass=0; fail=0
for i in 1 2 3 4 5; do
  SPX_PEER_TIMEOUT_S=60 SPX_SYNC_TIMEOUT_S=120 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29700 + i)) bench.py --gpus 4 --steps 30 --warmup 3 --config c4 --no-cpu-baseline --e2e-seconds 2 > gpurun_out/r2j_stress_$i.log 2>&1
  if [ $? -eq 0 ] && grep -q '"metric"' gpurun_out/r2j_stress_$i.log; then pass=$((pass+1)); else fail=$((fail+1)); fi
done
echo "C4 N=4 stress (final code): $pass passed, $fail failed"
