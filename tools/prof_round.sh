# ncu launch list of the default bench + one --set full capture per hot kernel (run under gpurun)
set -x
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch.log 2>&1; echo rc=$?
# k_round_tc: launch 32 = round 2 of a step (fold of the changed pixels), launch 39 = round 9
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_round_tc -s 31 -c 1 -o gpurun_out/round_tc -f $B > gpurun_out/ncu_tc.log 2>&1; echo rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_round_tc -s 38 -c 1 -o gpurun_out/round_tc_r9 -f $B > gpurun_out/ncu_tc9.log 2>&1; echo rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_encode -s 3 -c 1 -o gpurun_out/encode -f $B > gpurun_out/ncu_enc.log 2>&1; echo rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_finish_tc -s 20 -c 1 -o gpurun_out/finish_tc -f $B > gpurun_out/ncu_fin.log 2>&1; echo rc=$?
ls -la gpurun_out
