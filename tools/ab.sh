for v in 2 1 2 1; do SEGHDC_FLIST=$v timeout 300 python bench.py --no-cpu-baseline --steps 200 > gpurun_out/ab.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('FLIST=$v', d['value']/1e9, d['ms_per_step'], d['roofline']['avg_launch_ms'], d['e2e']['value']/1e9)"; done
SEGHDC_FLIST=2 timeout 200 python tools/round_times.py 1
