mkdir -p gpurun_out
timeout 600 python tools/tune_plans.py > gpurun_out/tune.log 2>&1; echo "EXIT $?" >> gpurun_out/tune.log
cp paper_1811_01532_b200/profiles/gemm_plans_b200.json gpurun_out/
timeout 1500 python -m pytest tests/test_bench_parity_gpu.py -m gpu -q -s > gpurun_out/parity.log 2>&1; echo "EXIT $?" >> gpurun_out/parity.log
timeout 600 python bench.py --no-cpu-baseline --breakdown > gpurun_out/bench_sacc.json 2> gpurun_out/bench_sacc.err
WAP_LIB_VARIANT=nosacc WAP_PLAN_CACHE=0 timeout 600 python bench.py --no-cpu-baseline --breakdown > gpurun_out/bench_nosacc.json 2> gpurun_out/bench_nosacc.err
timeout 600 python bench.py --no-cpu-baseline --breakdown > gpurun_out/bench_sacc2.json 2> gpurun_out/bench_sacc2.err
grep -E "decisions|passed|failed" gpurun_out/parity.log | tail; for f in sacc nosacc sacc2; do head -c 300 gpurun_out/bench_$f.json; echo; done
