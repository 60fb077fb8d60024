# closed-form variant, end-to-end ms per run: the cluster finish (default) vs the one-CTA one
for v in "" smem "" smem; do printf "finish=%-8s" "${v:-cluster}"; SEGHDC_CLOSED_FIN=$v timeout 300 python tools/closed_timing.py 2>&1 | tail -4 | tr '\n' ' '; echo; done
