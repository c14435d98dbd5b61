set -x
timeout 120 python scripts/trace_stage.py C2 > gpurun_out/tst_c2.json 2>&1
timeout 300 python scripts/trace_stage.py C3 > gpurun_out/tst_c3.json 2>&1
timeout 300 python scripts/trace_ed.py C3 > gpurun_out/ted_c3.json 2>&1
timeout 300 python scripts/trace_ed.py single8 > gpurun_out/ted_single8.json 2>&1
NS_STAGE_SPLIT=0 timeout 300 python bench.py --config C3 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/c3_nosplit.json 2>&1
