#!/bin/bash
# WY solve path / grid QR variants: parity tests and C4 timings under env variants (gpurun_out/)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -s --durations=0 -k "wy or C4 or n160 or owner or medium or tiled or variants" > gpurun_out/wy_tests.log 2>&1; echo "rc=$?" >> gpurun_out/wy_tests.log
run() { env "$@" timeout 600 python scripts/time_c4.py 4 2>&1 | tail -1 >> gpurun_out/wy_c4.jsonl; }
: > gpurun_out/wy_c4.jsonl
run NS_QR_CRIT=0
run NS_QR_CRIT=1
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_wy.json 2> gpurun_out/bench_wy.err
NS_QR_CRIT=1 timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_crit.json 2> gpurun_out/bench_crit.err
