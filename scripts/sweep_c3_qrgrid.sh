#!/bin/bash
# C3 grid-QR CTA count sweep (NS_QR_GRID; default 2n / 8 warps = 32) and the smem reservation
# that keeps eval/diff CTAs off the QR's SMs (NS_QR_RESERVE), QR beside eval/diff
mkdir -p gpurun_out/qg
run() { tag=$1; shift; env "$@" timeout 300 python bench.py --steps 20 --warmup 5 --no-extras --no-cpu-baseline > gpurun_out/qg/$tag.json 2> gpurun_out/qg/$tag.err; }
if [ "$1" = "2" ]; then
  run g32b NS_QR_GRID=32
  run g32_r0 NS_QR_GRID=32 NS_QR_RESERVE=0
  run g40b NS_QR_GRID=40
  run g40_r1 NS_QR_GRID=40 NS_QR_RESERVE=1
  run g48 NS_QR_GRID=48
  run g64 NS_QR_GRID=64
else
  for g in 16 24 32 40; do run g$g NS_QR_GRID=$g; done
fi
if [ "$1" = "3" ]; then
  run t128_g64_r0 NS_QR_THREADS=128 NS_QR_GRID=64 NS_QR_RESERVE=0
  run t128_g64_r1 NS_QR_THREADS=128 NS_QR_GRID=64 NS_QR_RESERVE=1
  run t128_g64_il NS_QR_THREADS=128 NS_QR_GRID=64 NS_QR_INTERLEAVE=1
  run g48b NS_QR_GRID=48
  run g32c NS_QR_GRID=32
fi
