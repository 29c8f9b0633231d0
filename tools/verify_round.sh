#!/bin/bash
# Fresh-box verification of the committed state: GPU suite, smoke, one bench line per config,
# the reference arm, and the launch list of the default bench command.
tag=${1:-r01s5}
o=gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > $o/${tag}_pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $o/${tag}_smoke.log 2>&1; echo "smoke rc=$?"
bash tools/bench_all.sh $tag
timeout 600 python bench.py > $o/plain_default.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $o/${tag}_launches_default.csv \
    python bench.py --no-cpu --no-e2e > $o/ncu_default.log 2>&1; echo "ncu rc=$?"
