# ncu launch list + one --set full capture of each round kernel variant (run under gpurun)
set -x
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_tc.csv $B > gpurun_out/ncu_launch_tc.log 2>&1; echo rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_round -s 30 -c 1 -o gpurun_out/round_tc -f $B > gpurun_out/ncu_tc.log 2>&1; echo rc=$?
SEGHDC_TC=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_round -s 30 -c 1 -o gpurun_out/round_imma -f $B > gpurun_out/ncu_imma.log 2>&1; echo rc=$?
SEGHDC_TC=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_imma.csv $B > gpurun_out/ncu_launch_imma.log 2>&1; echo rc=$?
ls -la gpurun_out
