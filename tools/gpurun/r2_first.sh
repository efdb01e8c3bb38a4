mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo "EXIT $?" >> gpurun_out/gputests.log
timeout 400 python bench.py > gpurun_out/bench_alexnet.json 2> gpurun_out/bench_alexnet.err
timeout 400 python bench.py --model vgg16 > gpurun_out/bench_vgg16.json 2> gpurun_out/bench_vgg16.err
tail -3 gpurun_out/gputests.log; cat gpurun_out/bench_alexnet.json | head -c 600; echo; head -c 600 gpurun_out/bench_vgg16.json
