mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 400 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gputests.log 2>&1; echo "EXIT $?" >> gpurun_out/gputests.log
tail -2 gpurun_out/smoke.log; tail -12 gpurun_out/gputests.log; head -c 300 gpurun_out/bench.json; echo; python -c "
import json; d=json.loads(open('gpurun_out/bench.json').read().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['vgg16']['value'], d['roofline']['kernel'], d['roofline']['kernel_ms'])"
