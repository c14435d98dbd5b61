#!/bin/bash
# after a QR-reflector change: the suite, then C2/C3/C4 timings, then this round's profiles
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -s --durations=10 > gpurun_out/tests.log 2>&1; echo "rc=$?" >> gpurun_out/tests.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
bash scripts/profile_r02.sh
