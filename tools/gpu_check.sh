for SM in "576,384" "576,256" "512,256" "448,320" "384,256"; do
 echo "smem=$SM $(KKT_POLL_NS=64 KKT_B_SMEM=$SM timeout 120 python tools/probe_kernels.py activsg10k 64 3 | cut -c1-100)"
done
for P in 0 32 128; do echo "poll=$P $(KKT_POLL_NS=$P KKT_B_SMEM=576,384 timeout 120 python tools/probe_kernels.py activsg10k 64 3 | cut -c1-100)"; done
