# L2-prefetch distance A/B for the N = 32 (C3) and split N = 64 (C4) layouts (per-round times)
for c in 3 4; do for pf in 8 0 4 16; do printf "C$c PF=$pf "; SEGHDC_PF=$pf timeout 300 python tools/round_times.py $c 6 | tail -1; done; done
