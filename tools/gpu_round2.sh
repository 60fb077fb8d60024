# GPU tests + C1/C2 bench lines (run under gpurun, one GPU)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/ -q -m gpu -x 2>&1 | tail -6
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/b_c1.json 2> gpurun_out/b_c1.err; echo c1 rc=$?
timeout 900 python bench.py --config 2 --steps 10 --no-cpu-baseline > gpurun_out/b_c2.json 2> gpurun_out/b_c2.err; echo c2 rc=$?
tail -2 gpurun_out/b_c2.err
for f in b_c1 b_c2; do python -c "
import json;d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1]);r=d['roofline'];e=d['e2e']
print('$f', '%.3e'%d['value'], d['ms_per_step'], r['avg_launch_ms'], r['frac'], 'e2e %.3e'%e['value'], 'ratio %.3f'%(e['value']/d['value']), d['gpu_launches'])"; done
