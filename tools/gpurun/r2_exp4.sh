mkdir -p gpurun_out
for cfg in "default:X=1" "notma:WAP_GEMM_NO_TMA_STORE=1" "epi2:WAP_LIB_VARIANT=epi2"; do
  name=${cfg%%:*}; envs=${cfg#*:}
  echo "== $name" >> gpurun_out/exp4.log
  env $envs timeout 300 python tools/gemm_times.py --model alexnet 2>&1 >> gpurun_out/exp4.log
done
cat gpurun_out/exp4.log
