# The 2d/4d/8d x N matrix of BASELINE.json's metric on one GPU (N = 2, 4, 8 come
# from the driver's scaling run): C4 and C5 at their own and the two swapped
# precisions (SURVEY 8(d) d.2 "precision-swapped"), the C3 headline, the T6 sweep.
set -x
mkdir -p gpurun_out
for K in 2 4 8; do
  timeout 900 python bench.py --config C5 --precision $K --steps 5 --warmup 3 > gpurun_out/matrix_c5_k$K.json 2> gpurun_out/matrix_c5_k$K.err
  timeout 900 python bench.py --config C4 --precision $K --steps 4 --warmup 2 > gpurun_out/matrix_c4_k$K.json 2> gpurun_out/matrix_c4_k$K.err
done
timeout 1200 python bench.py --sweep > gpurun_out/sweep_t6.json 2> gpurun_out/sweep_t6.err
