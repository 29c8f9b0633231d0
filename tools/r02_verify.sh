#!/bin/bash
# Round-2 verification on one B200: GPU suite, smoke, default bench line,
# the reference arm, then ncu of K1 at cfg3 (plain run first).
tag=${1:-r02v}
o=gpurun_out
free -g | head -2 > $o/${tag}_host.txt; nproc >> $o/${tag}_host.txt
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $o/${tag}_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $o/${tag}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $o/${tag}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python bench.py > $o/${tag}_bench.json 2> $o/${tag}_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > $o/${tag}_bench_ref.json 2> $o/${tag}_bench_ref.err; echo "ref rc=$?"
timeout 600 python bench.py --config cfg3 --steps 1 --warmup 3 --no-cpu --no-e2e --no-secondary > $o/${tag}_plain3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k1_tc_kernel" -s 2 -c 1 -o $o/${tag}_k1_cfg3 \
    python bench.py --config cfg3 --steps 1 --warmup 3 --no-cpu --no-e2e --no-secondary > $o/${tag}_ncu_f3.log 2>&1; echo "ncu rc=$?"
