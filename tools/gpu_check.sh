for v in 1 2 4; do echo "S=$v $(KKT_SWEEP_S=$v timeout 120 python tools/probe_kernels.py activsg10k 64 5 2>&1 | tail -1 | cut -c1-110)"; done
echo "nostage $(KKT_SWEEP_NOSTAGE=1 timeout 120 python tools/probe_kernels.py activsg10k 64 5 2>&1 | tail -1 | cut -c1-110)"
