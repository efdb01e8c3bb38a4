mkdir -p gpurun_out
for k in d_pool1 conv1; do
  echo "== $k"
  WAP_LIB_VARIANT=trace WAP_PLAN_CACHE=0 WAP_AUTOTUNE_FREE=1 timeout 200 python tools/gemm_trace.py --model alexnet --batch 128 --only $k 2>&1 | tail -5
done
for c in 8 16 32; do WAP_CHAIN_CHUNKS=$c WAP_AUTOTUNE=0 WAP_GEMM_CG=1 timeout 200 python tools/gemm_times.py --model alexnet --only d_pool1 2>&1 | grep d_pool1; done
