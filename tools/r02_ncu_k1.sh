#!/bin/bash
# ncu --set full of K1 at cfg3 (one launch).
tag=${1:-r02f}; o=gpurun_out
timeout 600 python bench.py --config cfg3 --steps 1 --warmup 3 --no-cpu --no-e2e --no-secondary > $o/${tag}_plain3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k1_tc_kernel" -s 2 -c 1 -o $o/${tag}_k1_cfg3 \
    python bench.py --config cfg3 --steps 1 --warmup 3 --no-cpu --no-e2e --no-secondary > $o/${tag}_ncu_f3.log 2>&1
echo "ncu full rc=$?"
