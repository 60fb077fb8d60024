# C1 (default bench) profiles on the final build (run under gpurun, one GPU)
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c1.csv $B > gpurun_out/ncu_launch_c1.log 2>&1; echo launches rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_round_tc -s 38 -c 1 -o gpurun_out/round_c1_r9 -f $B > gpurun_out/ncu_full_c1.log 2>&1; echo full rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_encode -s 3 -c 1 -o gpurun_out/encode_c1 -f $B > gpurun_out/ncu_enc_c1.log 2>&1; echo enc rc=$?
