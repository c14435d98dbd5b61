#!/bin/bash
# C5 (batched paths) launch-shape sweep: NS_BATCH_THREADS / NS_BATCH_CTAS / NS_BATCH_MINB
mkdir -p gpurun_out/c5
run() { tag=$1; shift; env "$@" timeout 300 python bench.py --config C5 --steps 10 --warmup 3 > gpurun_out/c5/$tag.json 2> gpurun_out/c5/$tag.err; }
run base
run minb2 NS_BATCH_MINB=2
run ctas3_minb2 NS_BATCH_CTAS=3 NS_BATCH_MINB=2
run ctas4_minb2 NS_BATCH_CTAS=4 NS_BATCH_MINB=2
run t128_ctas4_minb2 NS_BATCH_THREADS=128 NS_BATCH_CTAS=4 NS_BATCH_MINB=2
run t128_ctas6_minb2 NS_BATCH_THREADS=128 NS_BATCH_CTAS=6 NS_BATCH_MINB=2
run ctas1 NS_BATCH_CTAS=1
