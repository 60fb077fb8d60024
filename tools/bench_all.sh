# every config's bench line (run under gpurun, one GPU) into gpurun_out/bench_all/
mkdir -p gpurun_out/bench_all
timeout 900 python -m pytest tests/ -q -m gpu 2>&1 | tail -1
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/bench_all/c1.json 2> gpurun_out/bench_all/c1.err
for c in 0 2 3 4; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/bench_all/c$c.json 2> gpurun_out/bench_all/c$c.err
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_all/ref_c1.json 2> gpurun_out/bench_all/ref.err
for c in 0 1 2 3 4; do python -c "
import json;d=json.load(open('gpurun_out/bench_all/c$c.json'));r=d['roofline'];cb=d['cpu_baseline'] or {}
print('C$c', round(d['value']/1e9,3), round(d['ms_per_step'],3), r['kernel'], round(r['avg_launch_ms'],4), round(r['frac'],3), round(d['e2e']['value']/1e9,3), cb.get('value'), d['clocks'])"; done
