# same-box A/B of per-round kernel times: product build vs lib/<variant> (alternating), config $1, $2 rounds
V=${3:-old}
for i in 1 2; do
  printf "product  "; SEGHDC_PF=${PF:-0} timeout 300 python tools/round_times.py $1 $2 | tail -1
  printf "%-8s " $V; SEGHDC_PF=${PF:-0} SEGHDC_LIB=$PWD/paper_2303_12753_b200/lib/$V/libseghdc_b200.so timeout 300 python tools/round_times.py $1 $2 | tail -1
done
