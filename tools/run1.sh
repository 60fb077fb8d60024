set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -3
timeout 900 python -m pytest tests/ -q -m gpu -x 2>&1 | tail -8
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_tc.json 2> gpurun_out/bench_tc.err; echo rc=$?
SEGHDC_TC=0 timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_imma.json 2> gpurun_out/bench_imma.err; echo rc=$?
cat gpurun_out/bench_tc.json gpurun_out/bench_imma.json
tail -3 gpurun_out/bench_tc.err
