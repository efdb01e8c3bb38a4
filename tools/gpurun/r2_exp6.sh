mkdir -p gpurun_out
for cfg in "direct:X=1" "tmaplain:WAP_GEMM_TMA_STORE_PLAIN=1"; do
  name=${cfg%%:*}; envs=${cfg#*:}
  echo "== $name" >> gpurun_out/exp6.log
  env $envs timeout 300 python tools/gemm_times.py --model alexnet 2>&1 | grep -E "_w |total" >> gpurun_out/exp6.log
done
timeout 300 python -m pytest tests/test_gemm_gpu.py -m gpu -q -x 2>&1 | tail -2 >> gpurun_out/exp6.log
cat gpurun_out/exp6.log
