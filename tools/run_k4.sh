timeout 900 python -m pytest tests/ -q -m gpu -x 2>&1 | tail -3
for c in 3; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c$c.json 2>gpurun_out/bench_c$c.err; python -c "
import json;d=json.load(open('gpurun_out/bench_c$c.json'));r=d['roofline'];print('C$c', d['value']/1e9, d['ms_per_step'], r['kernel'], r['avg_launch_ms'], r['frac'])"; done
