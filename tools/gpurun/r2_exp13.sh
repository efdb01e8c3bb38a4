mkdir -p gpurun_out
timeout 120 python -m pytest tests/test_gemm_gpu.py -m gpu -q -x 2>&1 | tail -2
for i in 1 2 3; do timeout 60 python -m pytest tests/test_gemm_gpu.py -m gpu -q -x -k n64 2>&1 | tail -1; done
WAP_PLAN_CACHE=0 WAP_AUTOTUNE_FREE=1 timeout 240 python tools/hang_hunt.py --model alexnet --iters 3 > gpurun_out/hh.log 2>&1; echo "hang hunt EXIT $?"
WAP_AUTOTUNE=0 WAP_GEMM_CG=1 timeout 200 python tools/gemm_times.py --model alexnet 2>&1 | grep -E "bn= 64|total"
WAP_AUTOTUNE=0 WAP_GEMM_CG=1 timeout 200 python tools/gemm_times.py --model vgg16 2>&1 | grep -E "bn= 64|total"
