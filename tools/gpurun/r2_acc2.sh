mkdir -p gpurun_out
timeout 300 python tools/gemm_split_acc.py > gpurun_out/gemm_split_acc.log 2>&1
timeout 120 python tools/mc_create_probe.py > gpurun_out/mc_create.log 2>&1
nvidia-smi -q | grep -i -B2 -A6 "fabric" | head -30 >> gpurun_out/mc_create.log
cat gpurun_out/gemm_split_acc.log gpurun_out/mc_create.log
