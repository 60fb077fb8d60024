export SEGHDC_LIB=$PWD/paper_2303_12753_b200/lib/trace/libseghdc_b200.so
export SEGHDC_TRACE_ROUND=9
timeout 300 python tools/trace_tc.py 0 x 10 2>&1 | tail -30
echo ---- C1
timeout 300 python tools/trace_tc.py 1 x 10 2>&1 | tail -30
