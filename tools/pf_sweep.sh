# L2 prefetch distance sweep of the tcgen05 round kernel (run under gpurun)
for pf in 0 4 8 16 32; do echo "PF=$pf"; SEGHDC_PF=$pf timeout 120 python tools/trace_split.py 1024 | head -1; done
for pf in 0 8 16; do echo "C3 PF=$pf"; SEGHDC_PF=$pf timeout 300 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline | python -c "
import json,sys;d=json.loads(sys.stdin.read());r=d['roofline'];print(d['value']/1e9, d['ms_per_step'], r['avg_launch_ms'], r['frac'])"; done
