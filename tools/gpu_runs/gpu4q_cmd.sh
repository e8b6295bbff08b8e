export NCCL_DEBUG=WARN
mkdir -p gpurun_out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29514 tools/nccl_parity.py > gpurun_out/r2u_par_n4.log 2>&1
echo "parity N=4 rc=$?"; grep -v "^\[\|OMP_NUM\|^\*\*\*\|^NCCL version\|^\s*$" gpurun_out/r2u_par_n4.log | tail -1
SPX_NCCL_NONE=1 PARITY_CONFIGS=c3_tf1_bpz3_B8,c2_tf1_bpmp_B2M4,c4_unet_bpz2_B8 timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29800 tools/nccl_parity.py > gpurun_out/r2u_par_n8_on4.log 2>&1
echo "parity 8-on-4 rc=$?"; grep -v "^\[\|OMP_NUM\|^\*\*\*\|^\s*$" gpurun_out/r2u_par_n8_on4.log | tail -4
