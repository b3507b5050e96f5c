timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo tests=$? >> gpurun_out/gpu_tests.log
tail -2 gpurun_out/gpu_tests.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo bench=$?
tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['kernels'])"
timeout 1200 python tools/bench_configs.py activsg200 activsg2000 activsg10k activsg70k > gpurun_out/configs.jsonl 2>&1; echo cfg=$?
cat gpurun_out/configs.jsonl | cut -c1-400
