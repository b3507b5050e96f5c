timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_b_refactor$' -c 1 -o gpurun_out/prof_ref python tools/probe_kernels.py activsg10k 64 1 > gpurun_out/prof_ref.log 2>&1
echo ncu=$?
