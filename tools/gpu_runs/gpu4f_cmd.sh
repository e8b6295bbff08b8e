export NCCL_DEBUG=WARN
for N in 2 4; do
  SPX_CE_RS=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29510+N)) tools/nccl_parity.py > gpurun_out/r2f_par_n$N.log 2>&1
  echo "parity SPX_CE_RS=1 N=$N rc=$?"; grep -v "^\[\|OMP_NUM\|^\*\*\*\|^NCCL version\|^\s*$" gpurun_out/r2f_par_n$N.log | tail -7
done
for v in "SPX_CE_RS=1" "SPX_CE_RS=0"; do
  for c in c3 c5 c4; do
    st=30; [ "$c" = c3 ] && st=8
    env $v timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29720 bench.py --gpus 4 --steps $st --warmup 3 --config $c --no-cpu-baseline --e2e-seconds 5 > gpurun_out/r2f_${c}_n4_$v.log 2>&1
  done
done
SPX_CE_RS=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29730 bench.py --gpus 2 --steps 8 --warmup 3 --config c3 --no-cpu-baseline --e2e-seconds 5 > gpurun_out/r2f_c3_n2_SPX_CE_RS=1.log 2>&1
python tools/bench_summary.py gpurun_out/r2f_*.log
