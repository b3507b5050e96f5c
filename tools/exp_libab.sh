# usage: bash tools/exp_libab.sh TAG CONFIG B "ENV" ... — alternate ablib/old.so and ablib/new.so
T=$1; C=$2; B=$3; shift 3
L=paper_2401_13926_b200/libkktb200.so
cp $L /tmp/keep.so
for rep in 1 2; do
  for lib in ${LIBS:-old new}; do
    cp ablib/$lib.so $L
    for E in "$@"; do
      echo "== $lib $E" >> gpurun_out/${T}_libab.txt
      env $E timeout 600 python tools/probe_kernels.py $C $B 5 >> gpurun_out/${T}_libab.txt 2>&1
    done
  done
done
cp /tmp/keep.so $L
cat gpurun_out/${T}_libab.txt
