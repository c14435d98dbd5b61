#!/bin/bash
mkdir -p gpurun_out/ab
for cw in 8 4 2; do
  NS_STAGE2_CW=$cw NS_LEDGER=1 timeout 300 python bench.py --steps 20 --warmup 5 --no-extras --no-cpu-baseline > gpurun_out/ab/c3_cw$cw.json 2> gpurun_out/ab/c3_cw$cw.err
  NS_STAGE2_CW=$cw timeout 300 python bench.py --config C2 --steps 20 --warmup 5 --no-extras --no-cpu-baseline > gpurun_out/ab/c2_cw$cw.json 2> gpurun_out/ab/c2_cw$cw.err
done
NS_STAGE2_CW=4 timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "parity or staggered" > gpurun_out/ab/tests_cw4.log 2>&1; echo rc=$? >> gpurun_out/ab/tests_cw4.log
