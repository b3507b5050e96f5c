timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo bench=$?
tail -3 gpurun_out/bench.log | cut -c1-300
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo ref=$?
tail -1 gpurun_out/bench_ref.log | cut -c1-200
