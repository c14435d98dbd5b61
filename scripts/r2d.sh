set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -k "complex or batched or exponent or library or ledger or residual_sampling or owner_beta or n160" > gpurun_out/t3.log 2>&1; echo "rc=$?" >> gpurun_out/t3.log
timeout 300 python scripts/trace_batch.py 2 > gpurun_out/trace_batch_k2b.json 2>&1
NS_BATCH_MINB=1 timeout 300 python scripts/trace_batch.py 2 > gpurun_out/trace_batch_k2_minb1.json 2>&1
timeout 600 python scripts/time_c4.py 4 > gpurun_out/time_c4.json 2>&1
NS_QR_SMALLREGS=0 timeout 600 python scripts/time_c4.py 4 > gpurun_out/time_c4_bigregs.json 2>&1
