#!/bin/bash
# QR-variant check: parity tests of the WY / A0-alone paths and C3 timings under env variants (gpurun_out/)
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -s --durations=0 -k "wy or variants or medium or owner or tiled or C3_full or n160" > gpurun_out/wy_tests.log 2>&1; echo "rc=$?" >> gpurun_out/wy_tests.log
b() { tag=$1; shift; env "$@" timeout 600 python bench.py --steps 10 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/c3_$tag.json 2> gpurun_out/c3_$tag.err; }
b wym NS_WYM=1
b aug NS_WYM=0
b wym_st128 NS_WYM=1 NS_STAGE2_THREADS=128
b wym_qt256 NS_WYM=1 NS_QR_THREADS=256
timeout 300 python scripts/trace_batch.py 2 > gpurun_out/trace_batch_k2.json 2>&1
