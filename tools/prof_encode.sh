# encode kernel: write-bandwidth probe, timings, then one ncu --set full capture per config (run under gpurun)
mkdir -p gpurun_out/enc
./tools/probes/write_probe > gpurun_out/enc/write_probe.txt 2>&1; cat gpurun_out/enc/write_probe.txt
timeout 300 python tools/enc_time.py | tee gpurun_out/enc/enc_time.txt
for c in ${ENC_CONFIGS:-1 3}; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_encode -s 5 -c 1 -o gpurun_out/enc/encode_c$c -f python tools/enc_time.py $c > gpurun_out/enc/ncu_c$c.log 2>&1; echo ncu c$c rc=$?
  ncu -i gpurun_out/enc/encode_c$c.ncu-rep --page raw --csv > gpurun_out/enc/encode_c$c.raw.csv 2>/dev/null
done
