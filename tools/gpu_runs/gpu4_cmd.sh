export NCCL_DEBUG=WARN
# forward-progress stress: C4 B:4 with the defaults (side-stream GEMMs ON), 20 runs; a genuine GPU
# deadlock would now raise from the peer-barrier timeout (60 s) instead of hanging
pass=0; fail=0
for i in $(seq 1 20); do
  SPX_PEER_TIMEOUT_S=60 SPX_SYNC_TIMEOUT_S=120 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29600 + i)) \
    bench.py --gpus 4 --steps 30 --warmup 3 --config c4 --no-cpu-baseline --e2e-seconds 2 > gpurun_out/r2b_stress_c4_$i.log 2>&1
  rc=$?
  if [ $rc -eq 0 ] && grep -q '"metric"' gpurun_out/r2b_stress_c4_$i.log; then pass=$((pass+1)); else fail=$((fail+1)); echo "run $i rc=$rc"; grep "bench rank\|Error\|error" gpurun_out/r2b_stress_c4_$i.log | tail -8; fi
done
echo "C4 N=4 stress: $pass passed, $fail failed"
python tools/bench_summary.py gpurun_out/r2b_stress_c4_*.log | awk '{print $4}' | tr '\n' ' '; echo
bash tools/scale_runs.sh "4" "c5 c4" r2bn4
bash tools/_gpu4b_cmd.sh
