B="python tools/round_times.py 1"
timeout 600 ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg,sm__cycles_elapsed.avg,smsp__cycles_active.avg --clock-control none -k regex:k_round -c 20 --csv --log-file gpurun_out/ncu_rounds.csv $B > gpurun_out/ncu_rounds.log 2>&1; echo rc=$?
