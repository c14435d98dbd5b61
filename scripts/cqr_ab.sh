set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x > gpurun_out/cqr_parity.log 2>&1
NS_CQR_P=16 timeout 120 python scripts/trace_qr.py C2 > gpurun_out/tqr_c2_p16.json 2>&1
NS_CQR_P=8 timeout 120 python scripts/trace_qr.py C2 > gpurun_out/tqr_c2_p8.json 2>&1
for v in "1 16" "1 8" "0 8"; do
  set -- $v
  export NS_CQR=$1 NS_CQR_P=$2
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/cqr_c2_$1_$2.json 2>&1
done
