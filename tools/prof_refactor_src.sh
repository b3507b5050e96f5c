# usage: bash tools/prof_refactor_src.sh TAG — ncu --set full (with source counters) of the two
# batched refactor replay kernels at B = 64, then per-source-line summaries read back here
T=${1:-src}
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'k_b_refactor$|k_b_refactor_tma' -c 2 \
  -o gpurun_out/${T}_ref python tools/probe_kernels.py activsg10k 64 1 > gpurun_out/${T}_ref.log 2>&1
echo ncu=$?
ncu -i gpurun_out/${T}_ref.ncu-rep --page source --csv --print-source sass > gpurun_out/${T}_ref_sass.csv 2>/dev/null
ncu -i gpurun_out/${T}_ref.ncu-rep --page source --csv --print-source cuda > gpurun_out/${T}_ref_cuda.csv 2>/dev/null
ls -la gpurun_out/${T}_ref*
