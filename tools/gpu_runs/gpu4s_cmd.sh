export NCCL_DEBUG=WARN
mkdir -p gpurun_out
pass=0; fail=0
for i in 1 2 3 4; do
  SPX_PEER_TIMEOUT_S=60 SPX_SYNC_TIMEOUT_S=120 timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29700 + i)) bench.py --gpus 4 --steps 30 --warmup 3 --config c4 --no-cpu-baseline --e2e-seconds 2 > gpurun_out/r2w_stress_$i.log 2>&1
  if [ $? -eq 0 ] && grep -q '"metric"' gpurun_out/r2w_stress_$i.log; then pass=$((pass+1)); else fail=$((fail+1)); fi
  python tools/bench_summary.py gpurun_out/r2w_stress_$i.log | cut -c1-120
done
echo "C4 N=4 stress (final defaults): $pass passed, $fail failed"
