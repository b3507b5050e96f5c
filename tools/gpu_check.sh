echo "B1 $(timeout 120 python tools/probe_kernels.py activsg10k 1 5 2>&1 | tail -1 | cut -c1-110)"
timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
