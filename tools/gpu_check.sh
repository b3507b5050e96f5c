timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo tests=$? >> gpurun_out/gpu_tests.log
tail -2 gpurun_out/gpu_tests.log
for OV in 1 0; do for SP in 256 128; do
 echo "ov=$OV split=$SP $(KKT_B_OVERLAP=$OV KKT_B_SPLIT_NP=$SP timeout 120 python tools/probe_kernels.py activsg10k 64 3 | cut -c1-90)"
done; done
