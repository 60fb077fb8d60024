# where the round kernel's floor is (C1 and C3, per-round kernel times): product, no grid, no grid +
# no A stores into TMEM, no grid + no MMAs, no grid + neither (results meaningless; timing only)
L=$PWD/paper_2303_12753_b200/lib
for cfg in 1 3; do
  for v in "" nogrid exp_NOSTTM exp_NOMMA exp_NOSTTMNOMMA; do
    lib=${v:+$L/$v/libseghdc_b200.so}
    printf "config %s %-16s " $cfg "${v:-product}"; SEGHDC_LIB=$lib timeout 300 python tools/round_times.py $cfg 6 2>&1 | tail -1
  done
done
