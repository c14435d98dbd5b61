# A/B of the eval/diff convolution variants (NS_CONV_MODE, NS_CONV_TERMS)
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x > gpurun_out/ab_parity.log 2>&1
for cfg in "0 4" "0 2" "0 3" "1 4"; do
  set -- $cfg
  export NS_CONV_MODE=$1 NS_CONV_TERMS=$2
  python scripts/trace_ed.py single4 > gpurun_out/ab_single4_m$1_t$2.json 2>&1
  python scripts/trace_ed.py C2 > gpurun_out/ab_tc2_m$1_t$2.json 2>&1
  python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ab_c2_m$1_t$2.json 2>&1
done
for cfg in "0 4" "0 2" "1 4"; do
  set -- $cfg
  export NS_CONV_MODE=$1 NS_CONV_TERMS=$2
  python scripts/trace_ed.py single8 > gpurun_out/ab_single8_m$1_t$2.json 2>&1
  python bench.py --config C3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ab_c3_m$1_t$2.json 2>&1
done
