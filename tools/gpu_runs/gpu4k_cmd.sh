set -u
mkdir -p gpurun_out
for c in c3 c2 c4; do
  for n in 4; do
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29531 \
      tools/timeline.py --config $c --json gpurun_out/r2_tl_${c}_n$n.json > gpurun_out/r2_tl_${c}_n$n.log 2> gpurun_out/r2_tl_${c}_n$n.err
    echo "timeline $c N=$n rc=$?"
    head -1 gpurun_out/r2_tl_${c}_n$n.log | cut -c1-2500
  done
done
