for e in 32 64; do echo "70k E=$e $(KKT_B_TMA_E=$e timeout 300 python tools/probe_kernels.py activsg70k 64 2 2>&1 | tail -1 | cut -c1-110)"; done
echo "70k auto $(timeout 300 python tools/probe_kernels.py activsg70k 64 2 2>&1 | tail -1 | cut -c1-110)"
echo "10k auto $(timeout 300 python tools/probe_kernels.py activsg10k 64 3 2>&1 | tail -1 | cut -c1-110)"
timeout 900 python -m pytest tests/test_gpu_batch.py tests/test_gpu_scale.py -x -q -m gpu 2>&1 | tail -2
