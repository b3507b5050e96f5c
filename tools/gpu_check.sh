timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo tests=$? >> gpurun_out/gpu_tests.log
tail -2 gpurun_out/gpu_tests.log
timeout 120 python tools/probe_kernels.py activsg10k 64 3 --step
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/launches_step64.csv python tools/probe_kernels.py activsg10k 64 1 --step > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_step64.csv 2>/dev/null | head -30
