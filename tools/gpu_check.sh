for v in 1536 2048 3072 4096; do echo "rows=$v $(KKT_TAIL_ROWS=$v KKT_HEAD_ROWS=$v timeout 120 python tools/probe_kernels.py activsg10k 64 5 2>&1 | tail -1 | cut -c1-110)"; done
for v in 1536 3072; do echo "B1 rows=$v $(KKT_TAIL_ROWS=$v KKT_HEAD_ROWS=$v timeout 120 python tools/probe_kernels.py activsg10k 1 5 2>&1 | tail -1 | cut -c1-110)"; done
