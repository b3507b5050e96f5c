for st in 256 512 1024; do cp tools/libs_tmp/lib_rs$st.so paper_2401_13926_b200/libkktb200.so; touch paper_2401_13926_b200/libkktb200.so
echo "stage=$st $(timeout 120 python tools/probe_kernels.py activsg10k 1 5 | cut -c1-100)"
done
