mkdir -p gpurun_out
for cfg in "default:X=1" "pair3:WAP_LIB_VARIANT=pair3"; do
  name=${cfg%%:*}; envs=${cfg#*:}
  echo "== $name" >> gpurun_out/exp7.log
  env $envs WAP_AUTOTUNE=0 WAP_GEMM_CG=1 timeout 300 python tools/gemm_times.py --model alexnet 2>&1 | grep -E "bn= 64|total" >> gpurun_out/exp7.log
  env $envs WAP_AUTOTUNE=0 WAP_GEMM_CG=1 timeout 300 python tools/gemm_times.py --model vgg16 2>&1 | grep -E "bn= 64|total" >> gpurun_out/exp7.log
done
cat gpurun_out/exp7.log
