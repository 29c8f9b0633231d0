#!/bin/bash
# Final fresh-box verification (1 GPU): GPU suite, smoke, the default bench line
# and the reference arm. The ncu captures run in their own gpurun calls
# (tools/r02_ncu_list.sh, tools/r02_ncu_k1.sh): one ncu tool per call.
tag=${1:-r02f}
o=gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > $o/${tag}_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $o/${tag}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $o/${tag}_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 $o/${tag}_smoke.log
timeout 1500 python bench.py > $o/${tag}_bench.json 2> $o/${tag}_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > $o/${tag}_bench_ref.json 2> $o/${tag}_bench_ref.err; echo "ref rc=$?"
