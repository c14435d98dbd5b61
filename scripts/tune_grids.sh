set -x
python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -x > gpurun_out/gpu_tests.log 2>&1
for q in 16 32 64 148; do for s in 32 64 148; do
  NS_QR_GRID=$q NS_STAGE_GRID=$s python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/tune_c2_q${q}_s${s}.json 2>&1
done; done
python bench.py --config C3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3.json 2>&1
