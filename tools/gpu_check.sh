timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo tests=$? >> gpurun_out/gpu_tests.log
tail -3 gpurun_out/gpu_tests.log
for SP in 128 64 256 32 0; do
 echo "split=$SP $(KKT_B_SPLIT_NP=$SP timeout 120 python tools/probe_kernels.py activsg10k 64 3 | cut -c1-90)"
done
