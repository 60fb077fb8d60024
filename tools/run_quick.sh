# quick GPU check: gpu tests + bench (tc default and IMMA forced)
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -2
timeout 900 python -m pytest tests/ -q -m gpu -x 2>&1 | tail -8
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_tc.json 2> gpurun_out/bench_tc.err; echo rc=$?
python -c "import json;d=json.load(open('gpurun_out/bench_tc.json'));print('TC', d['value']/1e9, d['ms_per_step'], d['roofline']['avg_launch_ms'], d['roofline']['frac'], d['e2e']['value']/1e9)"
SEGHDC_TC=0 timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_imma.json 2> gpurun_out/bench_imma.err; echo rc=$?
python -c "import json;d=json.load(open('gpurun_out/bench_imma.json'));print('IMMA', d['value']/1e9, d['ms_per_step'], d['roofline']['avg_launch_ms'], d['roofline']['frac'], d['e2e']['value']/1e9)"
timeout 200 python tools/e2e_breakdown.py
