#!/bin/bash
# peer exchange on asymmetric grids (covers the row / column roles of 2x4)
o=gpurun_out
run() { timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $2 tools/grid_check.py; }
for s in "2 2x1" "4 1x4" "4 4x1"; do set -- $s
  RK_PEER=1 GRID_SHAPE=$2 run $1 $((29540 + $1)) > $o/shape_$2.log 2>&1; echo "$2 rc=$?"
  grep -o '"ok": [a-z]*' $o/shape_$2.log | head -1; grep -o '"exchange": "[a-z]*"' $o/shape_$2.log | sort | uniq -c
done
