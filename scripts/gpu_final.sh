set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/final_smi.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/final_gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/final_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1
timeout 400 python bench.py --steps 20 --warmup 5 > gpurun_out/final_c2.json 2>&1
timeout 400 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/final_c2_ref.json 2>&1
timeout 600 python bench.py --config C3 --steps 5 --warmup 3 > gpurun_out/final_c3.json 2>&1
timeout 300 python bench.py --config C1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/final_c1.json 2>&1
timeout 900 python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/final_c4.json 2>&1
timeout 900 python bench.py --config C4 --reuse-qr --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/final_c4_reuse.json 2>&1
timeout 900 python bench.py --config C5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/final_c5.json 2>&1
timeout 600 python bench.py --config C2 --driver --steps 5 --warmup 2 > gpurun_out/final_c2_driver.json 2>&1
timeout 900 python bench.py --config C3 --driver --steps 3 --warmup 1 > gpurun_out/final_c3_driver.json 2>&1
timeout 120 python scripts/trace_stage.py C2 > gpurun_out/final_tst_c2.json 2>&1
timeout 300 python scripts/trace_stage.py C3 > gpurun_out/final_tst_c3.json 2>&1
timeout 300 python scripts/trace_ed.py C3 > gpurun_out/final_ted_c3.json 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final_launches_c2.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final_launches_c3.csv python bench.py --config C3 --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
