# A/B of two library builds on the same box: ./tools/ab_lib.sh <script args...>
# runs `python tools/trace_split.py <args>` with the product build and with lib/old (alternating)
for i in 1 2; do
  for lib in "" "$PWD/paper_2303_12753_b200/lib/old/libseghdc_b200.so"; do
    SEGHDC_LIB=$lib timeout 300 python tools/trace_split.py "$@" 2>&1 | head -1 | sed "s#^#${lib:+old }#"
  done
done
