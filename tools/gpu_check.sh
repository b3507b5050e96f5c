timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
for r in 1 2; do echo "$(timeout 120 python tools/probe_kernels.py activsg10k 64 5 2>&1 | tail -1 | cut -c1-110)"; done
