export NCCL_DEBUG=WARN
N=4
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29510 tools/nccl_parity.py > gpurun_out/r2_par_n4.log 2>&1
echo "parity rc=$?"; grep -v "^\[\|OMP_NUM\|^\*\*\*" gpurun_out/r2_par_n4.log | tail -12
# forward-progress stress: C4 B:4 with the defaults (side-stream GEMMs ON), 20 runs
pass=0; fail=0
for i in $(seq 1 20); do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29600 + i)) \
    bench.py --gpus 4 --steps 30 --warmup 3 --config c4 --no-cpu-baseline --e2e-seconds 2 > gpurun_out/r2_stress_c4_$i.log 2>&1
  rc=$?
  if [ $rc -eq 0 ] && grep -q '"metric"' gpurun_out/r2_stress_c4_$i.log; then pass=$((pass+1)); else fail=$((fail+1)); echo "run $i rc=$rc"; tail -3 gpurun_out/r2_stress_c4_$i.log; fi
done
echo "C4 N=4 stress: $pass passed, $fail failed"
python tools/bench_summary.py gpurun_out/r2_stress_c4_*.log | awk '{print $4}' | tr '\n' ' '; echo
bash tools/scale_runs.sh "4" "c3 c2 c5" r2n4
