mkdir -p gpurun_out
for t in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_kernels.py > gpurun_out/sanitizer_$t.txt 2>&1; echo "EXIT $?" >> gpurun_out/sanitizer_$t.txt
done
WAP_AUTOTUNE=0 timeout 1800 python tools/measure_rank_steps.py --out gpurun_out/rank_steps.json > gpurun_out/rank_steps.log 2>&1; echo "EXIT $?" >> gpurun_out/rank_steps.log
for t in memcheck racecheck synccheck; do tail -4 gpurun_out/sanitizer_$t.txt; done
tail -5 gpurun_out/rank_steps.log
