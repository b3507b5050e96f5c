timeout 900 python bench.py > gpurun_out/r1j_bench.log 2>&1; echo bench=$?
