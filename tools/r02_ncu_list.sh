#!/bin/bash
# Launch list (first 400 launches) of the default bench command; per-launch times (cold, serialised).
tag=${1:-r02f}; o=gpurun_out
timeout 600 python bench.py --no-cpu --no-e2e --no-secondary --steps 3 --warmup 3 > $o/${tag}_plain_list.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
    --log-file $o/${tag}_launches_default.csv python bench.py --no-cpu --no-e2e --no-secondary --steps 3 --warmup 3 > $o/${tag}_ncu_default.log 2>&1
echo "ncu list rc=$?"
