mkdir -p gpurun_out
timeout 300 python tools/mc_probe.py > gpurun_out/mc_probe.log 2>&1
timeout 900 python tools/parity_diag.py --net alexnet --batch 128 > gpurun_out/diag_alex128.log 2>&1
timeout 300 python tools/parity_diag.py --net alexnet --batch 8 > gpurun_out/diag_alex8.log 2>&1
cat gpurun_out/mc_probe.log; cat gpurun_out/diag_alex128.log | head -80
