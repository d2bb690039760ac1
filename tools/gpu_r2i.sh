timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
SECONDS=0; timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; tail -3 gpurun_out/bench_full.err; echo "bench wall $SECONDS s"
python -c "
import json;d=json.load(open('gpurun_out/bench_full.json'))
print(d['value'], d['breakdown_ms'], d['roofline']['frac'], d['e2e'], d['saturation_events_per_step'], d['clocks'])
sw=d['subresults']['configs[4] sweep_8192_int8']
print({k:(round(v['value'],1), round(v['ms_per_step']*1e3,1)) for k,v in sw.items()})
"
