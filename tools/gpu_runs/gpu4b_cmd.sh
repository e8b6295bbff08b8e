export NCCL_DEBUG=WARN
echo "== peer all-reduce latency vs memory ordering (chain of 32 dependent all-reduces, graph replay)"
for n in 2 4; do for mb in 1 4 16; do for o in 0 1 2; do
  r=$(SPX_PEER_ORDER=$o timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29700 + n*10 + o)) tools/peer_bench.py --mb $mb 2>/dev/null | grep "{" | tail -1)
  echo "n=$n mb=$mb order=$o $r"
done; done; done
echo "== 8 ranks on 4 GPUs (two processes per GPU, peer-memory collectives only): the 8-member kernels"
SPX_NCCL_NONE=1 PARITY_CONFIGS=c3_tf1_bpz3_B8,c2_tf1_bpmp_B2M4,c4_unet_bpz2_B8,c5_tf1_bpmpz3emb_B2M2E2 timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29800 tools/nccl_parity.py > gpurun_out/r2_par_n8_on4.log 2>&1
echo "rc=$?"; grep -v "^\[\|OMP_NUM\|^\*\*\*" gpurun_out/r2_par_n8_on4.log | tail -15
