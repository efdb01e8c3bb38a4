WAP_LIB_VARIANT=psg3 timeout 120 python -m pytest tests/test_gemm_gpu.py -m gpu -q -x -k n64 2>&1 | tail -1
for cfg in "default:X=1" "psg3:WAP_LIB_VARIANT=psg3"; do
  name=${cfg%%:*}; envs=${cfg#*:}
  echo "== $name"
  env $envs WAP_AUTOTUNE=0 WAP_GEMM_CG=1 timeout 200 python tools/gemm_times.py --model alexnet 2>&1 | grep -E "bn= 64"
  env $envs WAP_AUTOTUNE=0 WAP_GEMM_CG=1 timeout 250 python tools/gemm_times.py --model vgg16 2>&1 | grep -E "bn= 64|total"
  env $envs WAP_PLAN_CACHE=0 WAP_AUTOTUNE_FREE=1 WAP_AUTOTUNE_LOG=1 timeout 250 python tools/gemm_times.py --model alexnet --only d_pool1 2>&1 | grep -E "autotune d_pool1"
done
