echo "10k $(timeout 120 python tools/probe_kernels.py activsg10k 64 5 2>&1 | tail -1 | cut -c1-110)"
echo "2000 $(timeout 120 python tools/probe_kernels.py activsg2000 64 5 2>&1 | tail -1 | cut -c1-110)"
echo "70k $(timeout 300 python tools/probe_kernels.py activsg70k 64 2 2>&1 | tail -1 | cut -c1-110)"
timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
