# usage: bash tools/exp_ab.sh TAG CONFIG B "ENV1" "ENV2" ... — batched refactor/solve time per env setting
T=$1; C=$2; B=$3; shift 3
for E in "$@"; do
  echo "== $E" >> gpurun_out/${T}_ab.txt
  env $E timeout 600 python tools/probe_kernels.py $C $B 5 >> gpurun_out/${T}_ab.txt 2>&1
done
cat gpurun_out/${T}_ab.txt
