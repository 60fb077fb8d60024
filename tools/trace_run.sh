export SEGHDC_LIB=$PWD/paper_2303_12753_b200/lib/trace/libseghdc_b200.so
timeout 300 python tools/trace_split.py 1024 4 2>&1 | tail -20
echo ----
timeout 300 python tools/trace_split.py 1024 3 2>&1 | tail -20
echo ---- untraced
unset SEGHDC_LIB
timeout 300 python tools/trace_split.py 1024 4 2>&1 | head -1
timeout 300 python tools/trace_split.py 1024 3 2>&1 | head -1
