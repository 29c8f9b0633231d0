#!/bin/bash
o=gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > $o/r01s5b_pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $o/r01s5b_smoke.log 2>&1; echo "smoke rc=$?"
for c in cfg4 cfg2 cfg3; do
  timeout 900 python bench.py --config $c > $o/r01s5b_bench_$c.json 2> $o/r01s5b_bench_$c.err; echo "$c rc=$?"
done
