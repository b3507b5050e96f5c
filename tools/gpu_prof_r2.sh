# round-2 evidence: ncu --set full of the top kernels on an IR-triggering B=64 step (k = 19,
# graph nodes profiled individually so the FGMRES kernels inside the conditional graph show),
# the launch list of the default bench command, and the single-system solve breakdown.
T=${1:-r2}
timeout 1500 ncu --set full --clock-control none --import-source on --graph-profiling node \
  -k regex:'k_b_refactor$|k_b_refactor2|k_b_refactor_tma|k_b_trsv_grid|k_trsv_blocked|k_b_spmv_row|k_b_dots|k_b_cgs|k_givens|k_b_expand_norms' \
  -c 16 -o gpurun_out/${T}_full python tools/step_probe.py activsg10k 64 19 1 > gpurun_out/${T}_full.log 2>&1
echo full=$?
python tools/ncu_traffic.py gpurun_out/${T}_full.ncu-rep gpurun_out/${T}_ncu_traffic.json > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/${T}_full.ncu-rep > gpurun_out/${T}_ncu_full_summary.txt 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --graph-profiling node --csv \
  --log-file gpurun_out/${T}_launches.csv python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-single --no-fixed --kernel-reps 1 > /dev/null 2>&1
echo launches=$?
python tools/launch_summary.py gpurun_out/${T}_launches.csv "ncu --graph-profiling node launch list of: python bench.py --steps 20 --warmup 5 (no cpu/single/fixed legs); cold-cache serialised launches: compare shares, not absolutes" > gpurun_out/${T}_launches_summary.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --graph-profiling node --csv \
  --log-file gpurun_out/${T}_single_launches.csv python tools/step_probe.py activsg10k 1 19 2 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/${T}_single_launches.csv "single-system k=19 step x2" > gpurun_out/${T}_single_launches_summary.txt
head -30 gpurun_out/${T}_launches_summary.txt; head -25 gpurun_out/${T}_single_launches_summary.txt; head -60 gpurun_out/${T}_ncu_full_summary.txt
