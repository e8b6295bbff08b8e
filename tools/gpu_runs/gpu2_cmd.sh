export NCCL_DEBUG=WARN
N=${N:-2}
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29510 tools/nccl_parity.py > gpurun_out/r2_par_n$N.log 2>&1
echo "parity rc=$?"; grep -v "^\[" gpurun_out/r2_par_n$N.log | tail -12
bash tools/scale_runs.sh "$N" "${CFGS:-c3 c2 c4 c5}" r2n$N
