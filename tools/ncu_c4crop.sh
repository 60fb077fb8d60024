# one --set full capture of the split-layout round kernel (K = 8, D = 16384, 1024^2 crop, the 4th launch)
# and of the C3-shape N = 32 kernel; raw pages dumped for the tensor-pipe metrics
mkdir -p gpurun_out/ncu
timeout 600 python tools/trace_split.py 1024 4 > /dev/null 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_round_tc -s 3 -c 1 \
  -o gpurun_out/ncu/c4crop -f python tools/trace_split.py 1024 4 > gpurun_out/ncu/c4crop.log 2>&1; echo rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_round_tc -s 3 -c 1 \
  -o gpurun_out/ncu/c3crop -f python tools/trace_split.py 1024 3 > gpurun_out/ncu/c3crop.log 2>&1; echo rc=$?
for r in c4crop c3crop; do ncu -i gpurun_out/ncu/$r.ncu-rep --page raw --csv > gpurun_out/ncu/$r.raw.csv 2>&1; done
ls -la gpurun_out/ncu
