# the checked build (-DSEGHDC_CHECKED device-side index checks) over the sanitizer cases (5 re-runs
# each) and the whole GPU test suite (run under gpurun, one GPU); log in gpurun_out/checked.log
export SEGHDC_LIB=$PWD/paper_2303_12753_b200/lib/checked/libseghdc_b200.so
mkdir -p gpurun_out
{ timeout 900 python tools/sanitize_cases.py; echo "cases rc=$?";
  timeout 1800 python -m pytest tests -q -m gpu 2>&1 | tail -4; echo "pytest rc=$?"; } > gpurun_out/checked.log 2>&1
cat gpurun_out/checked.log
