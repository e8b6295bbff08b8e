export NCCL_DEBUG=WARN
for v in "SPX_CE_AG=1" "SPX_CE_AG=0"; do
  for c in c3 c5; do
    st=30; [ "$c" = c3 ] && st=8
    env $v timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29720 bench.py --gpus 4 --steps $st --warmup 3 --config $c --no-cpu-baseline --e2e-seconds 5 > gpurun_out/r2e_${c}_n4_$v.log 2>&1
  done
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29730 bench.py --gpus 2 --steps 8 --warmup 3 --config c3 --no-cpu-baseline --e2e-seconds 5 > gpurun_out/r2e_c3_n2.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29731 bench.py --gpus 2 --steps 30 --warmup 3 --config c4 --no-cpu-baseline --e2e-seconds 5 > gpurun_out/r2e_c4_n2.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29732 bench.py --gpus 4 --steps 30 --warmup 3 --config c4 --no-cpu-baseline --e2e-seconds 5 > gpurun_out/r2e_c4_n4.log 2>&1
python tools/bench_summary.py gpurun_out/r2e_*.log
for s in "1024 512 512 64" "1024 1024 1024 64" "2048 1024 1024 64" "4096 2048 2048 32"; do timeout 300 python tools/gemm_chain.py $s; done
