# source-level ncu captures of the C2 kernels (one launch each, after warm-up)
for k in householder_qr stage_kernel evaldiff_jobs; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 -o gpurun_out/src_c2_$k python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_src_$k.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:householder_qr -s 2 -c 1 -o gpurun_out/src_c3_householder_qr python bench.py --config C3 --steps 1 --warmup 2 --no-cpu-baseline > gpurun_out/ncu_src_c3.log 2>&1
