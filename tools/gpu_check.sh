timeout 1500 python -m pytest tests/test_gpu_scale.py -x -q -m gpu --durations=10 > gpurun_out/gpu_scale.log 2>&1; echo scale=$? >> gpurun_out/gpu_scale.log
tail -20 gpurun_out/gpu_scale.log
