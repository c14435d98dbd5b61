#!/bin/bash
# Round check on the GPU box (outputs in gpurun_out/): the whole -m gpu suite and
# smoke(), the default bench line, the C3 launch list and FP64 counters.
# (compute-sanitizer is closed on this pool: see DESIGN.md section 10a)
mkdir -p gpurun_out
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider -s --durations=30 > gpurun_out/tests.log 2>&1; echo "rc=$?" >> gpurun_out/tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
bash scripts/gpu.sh launches C3
bash scripts/gpu.sh fp64 C3
