#!/bin/bash
# final check of a build (outputs in gpurun_out/): the whole -m gpu suite and smoke(),
# the default bench line, the C4 launch list and the C3 launch list
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -s --durations=10 > gpurun_out/tests.log 2>&1; echo "rc=$?" >> gpurun_out/tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
bash scripts/gpu.sh launches C4
bash scripts/gpu.sh launches C3
