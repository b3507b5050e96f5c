timeout 900 python -m pytest tests/test_gpu_batch.py -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo tests=$? >> gpurun_out/gpu_tests.log
tail -2 gpurun_out/gpu_tests.log
for M in 0 1; do for SC in 4 8; do for SP in 128 256; do
 echo "mode=$M sc=$SC split=$SP $(KKT_B_CT_MODE=$M KKT_B_CT_SC=$SC KKT_B_SPLIT_NP=$SP timeout 120 python tools/probe_kernels.py activsg10k 64 3 | cut -c1-90)"
done; done; done
