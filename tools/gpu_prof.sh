# round evidence: launch list of a short bench run + one --set full capture of the top kernels
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1c_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-single --kernel-reps 1 > gpurun_out/r1c_launches_run.log 2>&1
echo launches=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_b_refactor$|k_b_trsv_grid|k_trsv_blocked|k_b_spmv' -c 6 -o gpurun_out/r1c_full python tools/probe_kernels.py activsg10k 64 1 > gpurun_out/r1c_full.log 2>&1
echo full=$?
