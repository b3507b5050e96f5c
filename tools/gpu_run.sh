# usage: bash tools/gpu_run.sh TAG [pytest-args]  — GPU tests, smoke and the driver's bench on one B200
T=${1:-r2}; shift
P=${@:-tests}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${T}_gpu.txt 2>&1
timeout 2400 python -m pytest $P -q -m gpu --durations=20 > gpurun_out/${T}_gpu_tests.log 2>&1; echo tests=$? >> gpurun_out/${T}_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo smoke=$? >> gpurun_out/${T}_smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${T}_bench.log 2>&1; echo bench=$? >> gpurun_out/${T}_bench.log
tail -5 gpurun_out/${T}_gpu_tests.log; tail -2 gpurun_out/${T}_smoke.log; tail -c 600 gpurun_out/${T}_bench.log
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/${T}_bench_ref.log 2>&1; echo ref=$? >> gpurun_out/${T}_bench_ref.log
tail -c 400 gpurun_out/${T}_bench_ref.log
