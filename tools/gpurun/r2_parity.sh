mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_bench_parity_gpu.py tests/test_determinism_gpu.py -m gpu -q -s > gpurun_out/parity.log 2>&1; echo "EXIT $?" >> gpurun_out/parity.log
grep -E "step|decisions|passed|failed|Error" gpurun_out/parity.log | tail -30
