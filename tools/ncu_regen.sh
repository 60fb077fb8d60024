# ncu --set full of the C1 round kernel (round 9): the product build and the NOGRID experiment
# build (no grid stream: the upper bound of regenerating the HVs in the kernel)
mkdir -p gpurun_out/ncu
L=$PWD/paper_2303_12753_b200/lib
timeout 300 python tools/round_times.py 1 10 > /dev/null 2>&1
for v in product nogrid; do
  lib=""; [ $v = nogrid ] && lib=$L/nogrid/libseghdc_b200.so
  SEGHDC_LIB=$lib timeout 900 ncu --set full --clock-control none -k regex:k_round_tc -s 38 -c 1 -o gpurun_out/ncu/c1_$v -f \
    python tools/round_times.py 1 10 > gpurun_out/ncu/c1_$v.log 2>&1; echo "$v rc=$?"
  ncu -i gpurun_out/ncu/c1_$v.ncu-rep --page raw --csv > gpurun_out/ncu/c1_$v.raw.csv 2>&1
done
