mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gemm_gpu.py -m gpu -q -x > gpurun_out/t.log 2>&1; echo "EXIT $?" >> gpurun_out/t.log; tail -3 gpurun_out/t.log
if grep -q "EXIT 0" gpurun_out/t.log; then
for cfg in "onegroup:X=1" "twogroups:WAP_LIB_VARIANT=pair2g"; do
  name=${cfg%%:*}; envs=${cfg#*:}
  echo "== $name"
  env $envs WAP_AUTOTUNE=0 WAP_GEMM_CG=1 timeout 300 python tools/gemm_times.py --model alexnet 2>&1 | grep -E "bn= 64|total"
  env $envs WAP_AUTOTUNE=0 WAP_GEMM_CG=1 timeout 300 python tools/gemm_times.py --model vgg16 2>&1 | grep -E "bn= 64|total"
done
fi
