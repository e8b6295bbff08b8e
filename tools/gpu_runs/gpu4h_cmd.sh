export NCCL_DEBUG=WARN
SPX_PEER_PREBARRIER=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29514 tools/nccl_parity.py > gpurun_out/r2h_par_n4.log 2>&1
echo "parity prebarrier N=4 rc=$?"; grep -v "^\[\|OMP_NUM\|^\*\*\*\|^NCCL version\|^\s*$" gpurun_out/r2h_par_n4.log | tail -2
for v in "SPX_PEER_PREBARRIER=1" "SPX_PEER_PREBARRIER=0"; do
  for c in c3 c5 c4; do
    st=30; [ "$c" = c3 ] && st=8
    env $v timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29720 bench.py --gpus 4 --steps $st --warmup 3 --config $c --no-cpu-baseline --e2e-seconds 3 > gpurun_out/r2h_${c}_n4_$v.log 2>&1
  done
done
SPX_PEER_PREBARRIER=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29730 bench.py --gpus 2 --steps 8 --warmup 3 --config c3 --no-cpu-baseline --e2e-seconds 3 > gpurun_out/r2h_c3_n2_SPX_PEER_PREBARRIER=1.log 2>&1
python tools/bench_summary.py gpurun_out/r2h_*.log
