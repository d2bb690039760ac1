timeout 600 python -m pytest tests/test_gpu_contracts.py tests/test_multirank.py -x -q 2>&1 | tail -2
SECONDS=0; timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; tail -3 gpurun_out/bench_full.err; echo "bench wall $SECONDS s"
python -c "
import json;d=json.load(open('gpurun_out/bench_full.json'))
print(d['value'], d['breakdown_ms'], d['roofline']['frac'], d['e2e'], d['cpu_baseline'], d['saturation_events_per_step'], d['clocks'])
for k,v in d['subresults'].items(): print(k, json.dumps(v)[:600])
"
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 | cut -c1-400
