#!/bin/bash
o=gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > $o/r01s5c_pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $o/r01s5c_smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > $o/r01s5c_bench_default.json 2> $o/r01s5c_bench_default.err; echo "bench rc=$?"
timeout 600 python bench.py --config cfg1 > $o/r01s5c_bench_cfg1.json 2> $o/r01s5c_bench_cfg1.err; echo "cfg1 rc=$?"
timeout 600 python bench.py --config cfg5 > $o/r01s5c_bench_cfg5.json 2> $o/r01s5c_bench_cfg5.err; echo "cfg5 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"sp_gram_tc_k" -s 4 -c 1 -o $o/r01s5c_gram32_k32m \
  python tools/phase_split.py k32m > $o/ncu_g32.log 2>&1; echo "ncu rc=$?"
