#!/bin/bash
# ncu summaries of this round's kernels (outputs in gpurun_out/): the C3 headline's QR,
# the C4 critical-chain QR and WY stage, the C4 launch list; then the 2d/4d/8d matrix.
bash scripts/gpu.sh full C3 householder_qr_kernel
bash scripts/gpu.sh full C4 householder_qr_crit_kernel
bash scripts/gpu.sh full C4 stage_wy_kernel
bash scripts/gpu.sh launches C4
bash scripts/matrix.sh
