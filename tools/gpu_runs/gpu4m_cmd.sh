export NCCL_DEBUG=WARN
mkdir -p gpurun_out
run() {  # tag config env...
  tag=$1; c=$2; shift 2
  st=30; [ "$c" = c3 ] && st=10
  env "$@" timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 4 --steps $st --warmup 5 --config $c --no-cpu-baseline > gpurun_out/r2m_${tag}.log 2>&1
  echo "$tag $*: $(python tools/bench_summary.py gpurun_out/r2m_${tag}.log | cut -c1-260)"
}
run c3_hoist0 c3 SPX_HOIST_COLL=0
run c3_hoist1 c3 SPX_HOIST_COLL=1
run c3_cers c3 SPX_CE_RS=1
run c3_ob32 c3 SPX_PEER_OFFCRIT_BLOCKS=32
run c3_ob64 c3 SPX_PEER_OFFCRIT_BLOCKS=64
run c3_cers_h0 c3 SPX_CE_RS=1 SPX_HOIST_COLL=0
run c2_hoist0 c2 SPX_HOIST_COLL=0
run c5_hoist0 c5 SPX_HOIST_COLL=0
run c5_cers c5 SPX_CE_RS=1
