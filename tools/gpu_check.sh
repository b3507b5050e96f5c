timeout 900 python bench.py > gpurun_out/r1k_bench2.log 2>&1; echo bench=$?
timeout 900 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
