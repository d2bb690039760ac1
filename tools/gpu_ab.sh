# A/B of K4 tile shapes in one session: alternate runs, K4 graph-timed ms
for i in 1 2 3; do
for nb in 3 2; do
FQG_GEMM_NB=$nb timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-subresults --e2e-steps 1 > gpurun_out/ab.json; python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('NB$nb', round(d['value'],1), round(d['breakdown_ms']['gemm_K4']*1e3,2), round(d['breakdown_ms']['K1_K4_graph']*1e3,2))"
done; done
