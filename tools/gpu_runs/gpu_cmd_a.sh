SPX_H3_DYNAMIC=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "h3 or gemm" 2>&1 | tail -2
SPX_H3_DYNAMIC=1 timeout 900 python -m pytest tests/test_config_parity.py -q -m gpu -x 2>&1 | tail -2
for v in "SPX_H3_DYNAMIC=0" "SPX_H3_DYNAMIC=1" "SPX_H3_DYNAMIC=1 SPX_PIECES_ONLY=0" "SPX_H3_DYNAMIC=0 SPX_PIECES_ONLY=0"; do
  env $v timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-seconds 5 > gpurun_out/r2_c3_var.json 2>/dev/null
  echo "variant [$v]: $(python -c "import json; d=json.load(open('gpurun_out/r2_c3_var.json')); print(round(d['value']), round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value']), d['clocks']['sm_mhz'], d['roofline']['step_ms_by_class'], round(d['roofline']['frac'],3), round(d['streaming_roofline']['frac'],3))")"
done
