#!/bin/bash
# Round check on the GPU box: the whole -m gpu suite (+ smoke), then compute-sanitizer
# racecheck / synccheck / memcheck on C1 / C2 / a C5 batch of 8 (outputs in gpurun_out/)
mkdir -p gpurun_out
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider -s --durations=30 > gpurun_out/tests.log 2>&1; echo "rc=$?" >> gpurun_out/tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
for tool in racecheck synccheck memcheck; do
  for C in C1 C2; do
    timeout 420 compute-sanitizer --tool $tool --print-limit 20 python scripts/one_step.py $C 0 > gpurun_out/sanitize_${tool}_$C.log 2>&1
    echo "rc=$?" >> gpurun_out/sanitize_${tool}_$C.log
  done
  timeout 420 compute-sanitizer --tool $tool --print-limit 20 python scripts/one_step.py C5 0 2 8 > gpurun_out/sanitize_${tool}_C5b8.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitize_${tool}_C5b8.log
done
