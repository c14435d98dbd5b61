timeout 900 ncu --set full --clock-control none --import-source on -k regex:evaldiff_jobs -s 2 -c 1 -o gpurun_out/src_c3_evaldiff python bench.py --config C3 --steps 1 --warmup 2 --no-cpu-baseline > gpurun_out/ncu_c3_ed.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stage2 -s 2 -c 1 -o gpurun_out/src_c3_stage2 python bench.py --config C3 --steps 1 --warmup 2 --no-cpu-baseline > gpurun_out/ncu_c3_st.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/torchrun_n1.json 2> gpurun_out/torchrun_n1.err
python bench.py --no-cpu-baseline > gpurun_out/bench_c2.json 2>&1
python bench.py --config C3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3.json 2>&1
