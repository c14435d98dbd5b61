set -x
mkdir -p gpurun_out
bash scripts/gpu.sh full C5 batched_step
bash scripts/gpu.sh full C3 evaldiff_jobs
bash scripts/gpu.sh full C3 stage2
bash scripts/gpu.sh launches C3
bash scripts/gpu.sh fp64 C2
bash scripts/gpu.sh launches C4
du -sh gpurun_out
