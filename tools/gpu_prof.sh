# round-1 evidence (r1l): tests, smoke, bench, reference arm, launch list, ncu --set full of the top kernels
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/r1l_gpu_tests.log 2>&1; echo tests=$? >> gpurun_out/r1l_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1l_smoke.log 2>&1; echo smoke=$? >> gpurun_out/r1l_smoke.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_b_refactor$|k_b_refactor_tma|k_b_trsv_grid|k_trsv_blocked|k_b_spmv' -c 7 -o gpurun_out/r1l_full python tools/probe_kernels.py activsg10k 64 1 --step > gpurun_out/r1l_full.log 2>&1
echo full=$?
python tools/ncu_traffic.py gpurun_out/r1l_full.ncu-rep profiles/r1l_ncu_traffic.json > /dev/null 2>&1; cp profiles/r1l_ncu_traffic.json gpurun_out/ 2>/dev/null
timeout 900 python bench.py > gpurun_out/r1l_bench.log 2>&1; echo bench=$?
timeout 900 python bench.py --impl reference > gpurun_out/r1l_bench_ref.log 2>&1; echo ref=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1l_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-single --kernel-reps 1 > /dev/null 2>&1
echo launches=$?
tail -2 gpurun_out/r1l_gpu_tests.log; tail -1 gpurun_out/r1l_smoke.log
