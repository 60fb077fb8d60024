# C3/C4 profiles (run under gpurun, one GPU): launch lists of one bench step and a --set full
# capture of each config's round kernel
for c in 3 4; do
  B="python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline"
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_c$c.csv $B > gpurun_out/ncu_launch_c$c.log 2>&1; echo launches c$c rc=$?
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_round_tc -s 12 -c 1 -o gpurun_out/round_c$c -f $B > gpurun_out/ncu_full_c$c.log 2>&1; echo full c$c rc=$?
done
