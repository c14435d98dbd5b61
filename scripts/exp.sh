#!/bin/bash
mkdir -p gpurun_out
timeout 2000 python -m pytest tests -m gpu -q -p no:cacheprovider -s -k "C3_full or C3_sampled" --timeout 900 --timeout_method=thread > gpurun_out/c3tests.log 2>&1; echo "rc=$?" >> gpurun_out/c3tests.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/c3_default.json 2> gpurun_out/c3_default.err
timeout 600 python bench.py --config C5 --steps 5 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/c5_256.json 2> gpurun_out/c5_256.err
NS_BATCH_THREADS=128 NS_BATCH_CTAS=4 timeout 600 python bench.py --config C5 --steps 5 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/c5_128.json 2> gpurun_out/c5_128.err
bash scripts/gpu.sh launches C3
