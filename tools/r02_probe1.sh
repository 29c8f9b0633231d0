#!/bin/bash
# Round-2 first probe: cfg3 bench line, cfg3 launch list, ncu --set full of K1<32> at cfg3.
o=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $o/r02p1_smi.txt 2>&1
timeout 600 python bench.py --config cfg3 --steps 20 --warmup 3 --no-cpu --no-e2e > $o/r02p1_bench_cfg3.log 2>&1; echo "bench rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $o/r02p1_launches_cfg3.csv \
    python bench.py --config cfg3 --steps 2 --warmup 3 --no-cpu --no-e2e > $o/r02p1_ncu_l3.log 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k1_tc_kernel" -s 2 -c 1 -o $o/r02p1_k1_cfg3 \
    python bench.py --config cfg3 --steps 1 --warmup 3 --no-cpu --no-e2e > $o/r02p1_ncu_f3.log 2>&1; echo "ncu full rc=$?"
