for c in 2 4 6 8; do echo "cap=$c $(KKT_SMALL_LEVELS=$c timeout 120 python tools/probe_kernels.py activsg10k 64 5 2>&1 | tail -1 | cut -c1-110)"; done
for c in 2 8; do echo "2000 cap=$c $(KKT_SMALL_LEVELS=$c timeout 120 python tools/probe_kernels.py activsg2000 64 5 2>&1 | tail -1 | cut -c1-110)"; done
for c in 2 8; do echo "B1 cap=$c $(KKT_SMALL_LEVELS=$c timeout 120 python tools/probe_kernels.py activsg10k 1 5 2>&1 | tail -1 | cut -c1-110)"; done
