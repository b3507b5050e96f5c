timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo tests=$? >> gpurun_out/gpu_tests.log
tail -2 gpurun_out/gpu_tests.log
timeout 120 python tools/trace_grid.py activsg10k 1
timeout 120 python tools/trace_grid.py activsg10k 64
timeout 120 python tools/probe_kernels.py activsg10k 1 3
timeout 120 python tools/probe_kernels.py activsg10k 64 3 --step
