# usage: bash tools/exp_refactor_split.sh TAG — batched refactor kernels at B = 32/64/128, with
# and without dependency waits (KKT_NO_RESET=1 keeps the previous factors published), per
# kernel from the ncu launch list (serialised, so compare between rows, not absolutes)
T=${1:-exp}
for B in 32 64 128; do
  for NR in 0 1; do
    if [ $NR = 1 ]; then export KKT_NO_RESET=1; else unset KKT_NO_RESET; fi
    timeout 600 python tools/probe_kernels.py activsg10k $B 3 >> gpurun_out/${T}_probe.txt 2>&1
    timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:'k_b_refactor' \
      --log-file gpurun_out/${T}_B${B}_nr${NR}.csv python tools/probe_kernels.py activsg10k $B 2 > /dev/null 2>&1
    echo "B=$B no_reset=$NR"; python tools/launch_summary.py gpurun_out/${T}_B${B}_nr${NR}.csv "B=$B nr=$NR" | head -8
  done
done
unset KKT_NO_RESET
cat gpurun_out/${T}_probe.txt
