# upper bound for regenerating the pixel HVs inside the round kernel: the NOGRID experiment build
# (no TMA stream, no shared-memory reads; A words from a hash) vs the product build, per round
for cfg in 1 0 3; do
  echo "config $cfg product:"; timeout 300 python tools/round_times.py $cfg 10
  echo "config $cfg NOGRID:"; SEGHDC_LIB=$PWD/paper_2303_12753_b200/lib/nogrid/libseghdc_b200.so timeout 300 python tools/round_times.py $cfg 10
done
