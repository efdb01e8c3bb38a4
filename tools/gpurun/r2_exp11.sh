mkdir -p gpurun_out
WAP_LIB_VARIANT=pairss timeout 300 python -m pytest tests/test_gemm_gpu.py -m gpu -q -x -k n64 2>&1 | tail -2
for cfg in "ts:X=1" "ss:WAP_LIB_VARIANT=pairss"; do
  name=${cfg%%:*}; envs=${cfg#*:}
  echo "== $name"
  env $envs WAP_AUTOTUNE=0 WAP_GEMM_CG=1 timeout 300 python tools/gemm_times.py --model alexnet 2>&1 | grep -E "bn= 64|total"
  env $envs WAP_AUTOTUNE=0 WAP_GEMM_CG=1 timeout 300 python tools/gemm_times.py --model vgg16 2>&1 | grep -E "bn= 64|total"
done
