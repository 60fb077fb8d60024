# build and run the C++ drop-in bench (reference CLI protocol) on every config (under gpurun)
set -e
L=$PWD/paper_2303_12753_b200/lib; W=$PWD/workloads/lib
g++ -std=c++20 -O2 -Iinclude tools/cpp_bench.cpp -o /tmp/cpp_bench -L$L -lseghdc_b200 -L$W -lseghdc_synth \
  -L/usr/local/cuda/lib64 -lcudart -Wl,-rpath,$L -Wl,-rpath,$W -Wl,-rpath,/usr/local/cuda/lib64
for c in 0 1 3 4; do timeout 300 /tmp/cpp_bench $c ${REPEATS:-20}; done
