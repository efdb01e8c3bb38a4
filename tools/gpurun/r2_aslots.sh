mkdir -p gpurun_out
for v in nosacc nosacca2; do
  WAP_LIB_VARIANT=$v WAP_PLAN_CACHE=0 WAP_AUTOTUNE_FREE=1 timeout 600 python bench.py --model alexnet --no-cpu-baseline --breakdown > gpurun_out/bench_$v.json 2> gpurun_out/bench_$v.err
done
WAP_PLAN_CACHE=0 WAP_AUTOTUNE_FREE=1 timeout 600 python bench.py --model alexnet --no-cpu-baseline --breakdown > gpurun_out/bench_sacc_free.json 2> gpurun_out/bench_sacc_free.err
for t in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_kernels.py > gpurun_out/sanitizer_$t.txt 2>&1; echo "EXIT $?" >> gpurun_out/sanitizer_$t.txt
done
for v in nosacc nosacca2 sacc_free; do head -c 200 gpurun_out/bench_$v.json; echo; done
for t in memcheck racecheck synccheck; do tail -4 gpurun_out/sanitizer_$t.txt; done
