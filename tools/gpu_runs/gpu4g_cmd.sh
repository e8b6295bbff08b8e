export NCCL_DEBUG=WARN
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "h3 or gemm" 2>&1 | tail -2
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-seconds 5 > gpurun_out/r2g_c3_n1.log 2>&1
for N in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29720+N)) bench.py --gpus $N --steps 8 --warmup 3 --config c3 --no-cpu-baseline --e2e-seconds 5 > gpurun_out/r2g_c3_n$N.log 2>&1
done
python tools/bench_summary.py gpurun_out/r2g_*.log
echo "== 8 ranks on 4 GPUs, current defaults (copy-engine gathers from 16 MB)"
SPX_NCCL_NONE=1 PARITY_CONFIGS=c3_tf1_bpz3_B8,c2_tf1_bpmp_B2M4,c4_unet_bpz2_B8 timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29800 tools/nccl_parity.py > gpurun_out/r2g_par_n8_on4.log 2>&1
echo "rc=$?"; grep -v "^\[\|OMP_NUM\|^\*\*\*\|^\s*$" gpurun_out/r2g_par_n8_on4.log | tail -6
