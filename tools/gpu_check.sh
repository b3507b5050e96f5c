timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
for r in 1 2; do timeout 600 python bench.py --no-single --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['kernels']['spmv']['ms'])"; done
