# round-2 measurement pass (under gpurun, one GPU): every config's bench line, then the ncu
# launch list of the default bench command and a --set full capture of each config's round
# kernel (traffic per launch -> profiles/round2_traffic_c*.json via tools/ncu_summary.py)
mkdir -p gpurun_out/r2
timeout 600 python bench.py > gpurun_out/r2/c1.json 2> gpurun_out/r2/c1.err; echo c1 rc=$?
for c in 0 2 3 4; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/r2/c$c.json 2> gpurun_out/r2/c$c.err; echo c$c rc=$?
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2/ref_c1.json 2> gpurun_out/r2/ref.err; echo ref rc=$?
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/r2/launches_c1.csv $B > gpurun_out/r2/ncu_launch_c1.log 2>&1; echo launches rc=$?
for c in 1 0 3 4; do
  B="python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline"
  S=$([ $c = 1 ] && echo 38 || ([ $c = 0 ] && echo 38 || echo 12))
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_round_tc -s $S -c 1 -o gpurun_out/r2/round_c$c -f $B > gpurun_out/r2/ncu_full_c$c.log 2>&1; echo full c$c rc=$?
  ncu -i gpurun_out/r2/round_c$c.ncu-rep --page raw --csv > gpurun_out/r2/round_c$c.raw.csv 2>/dev/null
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_encode -s 3 -c 1 -o gpurun_out/r2/encode_c1 -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r2/ncu_enc.log 2>&1; echo enc rc=$?
ncu -i gpurun_out/r2/encode_c1.ncu-rep --page raw --csv > gpurun_out/r2/encode_c1.raw.csv 2>/dev/null
ls gpurun_out/r2
