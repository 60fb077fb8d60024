SEGHDC_LIB=$PWD/paper_2303_12753_b200/lib/trace/libseghdc_b200.so timeout 200 python tools/trace_tc.py 1
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_round -s 30 -c 1 -o gpurun_out/round_tc -f $B > gpurun_out/ncu_tc.log 2>&1; echo rc=$?
