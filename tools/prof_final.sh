# Final measurement pass of a round (run under gpurun, one GPU). Everything lands in
# gpurun_out/final/ as small text files (the ncu reports are summarised on the box and deleted):
#   checked.log          the -DSEGHDC_CHECKED build over the sanitizer cases and the whole GPU suite
#   c<config>.json       bench lines; ref_c1.json the reference arm
#   launches_c1.csv      ncu launch list of the default bench command
#   traffic_c<config>.*  ncu --set full of the round kernel (DRAM bytes per launch + summary)
#   encode_c<config>.md  ncu --set full of the encode kernel
#   cpp_bench.jsonl      the C++ drop-in caller (reference CLI bench protocol)
#   closed.jsonl         the closed-form variant end to end
O=gpurun_out/final; mkdir -p $O
bash tools/checked_run.sh > /dev/null 2>&1; cp gpurun_out/checked.log $O/checked.log; tail -3 $O/checked.log
timeout 600 python bench.py > $O/c1.json 2> $O/c1.err; echo c1 rc=$?
for c in 0 2 3 4; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 > $O/c$c.json 2> $O/c$c.err; echo c$c rc=$?
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/ref_c1.json 2> $O/ref.err; echo ref rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
  --log-file $O/launches_c1.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch_c1.log 2>&1; echo launches rc=$?
for c in 1 0 3 4; do
  S=$([ $c = 1 ] && echo 38 || ([ $c = 0 ] && echo 38 || echo 12))
  timeout 900 ncu --set full --clock-control none -k regex:k_round_tc -s $S -c 1 -o /tmp/round_c$c -f \
    python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_full_c$c.log 2>&1; echo full c$c rc=$?
  python tools/ncu_summary.py traffic /tmp/round_c$c.ncu-rep $O/traffic_c$c.json $c
done
for c in 1 3 4; do
  timeout 600 ncu --set full --clock-control none -k regex:k_encode -s 5 -c 1 -o /tmp/encode_c$c -f python tools/enc_time.py $c > $O/ncu_enc_c$c.log 2>&1; echo enc c$c rc=$?
  python tools/ncu_summary.py kernel /tmp/encode_c$c.ncu-rep $O/encode_c$c.md > /dev/null
done
timeout 300 python tools/enc_time.py > $O/enc_time.txt 2>&1
REPEATS=20 bash tools/cpp_bench.sh > $O/cpp_bench.jsonl 2> $O/cpp_bench.err; echo cpp rc=$?
timeout 600 python tools/closed_timing.py > $O/closed.jsonl 2> $O/closed.err; echo closed rc=$?
for c in 0 1 2 3 4; do python -c "
import json;d=json.load(open('$O/c$c.json'));r=d['roofline'];cb=d['cpu_baseline'] or {}
print('C$c', round(d['value']/1e9,3), round(d['ms_per_step'],3), round(r['avg_launch_ms'],4), round(r['frac'],3), round(d['e2e']['value']/1e9,3), cb.get('value'), d['clocks'])"; done
ls -la $O | head -40
