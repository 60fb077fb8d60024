# round-end style run: GPU tests, smoke, default bench, reference arm (run under gpurun)
set -x
timeout 900 python -m pytest tests/ -q -m gpu -x 2>&1 | tail -3
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench rc=$?
cat gpurun_out/bench_default.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref rc=$?
cat gpurun_out/bench_ref.json
