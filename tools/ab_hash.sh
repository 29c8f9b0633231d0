#!/bin/bash
# Same-input A/B of two library builds: factor hashes after 20 iterations (must match
# bit for bit when a change keeps the arithmetic) and graph-replayed ms/iteration.
# old = paper_2202_09512_b200/librescal_b200_head.so (build of the last commit).
cfgs=${1:-"cfg1 cfg2 k32s cfg5 k48 k64"}
for cfg in $cfgs; do
  for lib in old new; do
    if [ $lib = old ]; then L=$PWD/paper_2202_09512_b200/librescal_b200_head.so; else L=$PWD/paper_2202_09512_b200/librescal_b200.so; fi
    RK_LIB_PATH=$L timeout 300 python tools/k2af_check.py $cfg 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$cfg', '$lib', d['hash_track0'], d['hash_track1'], round(d['ms_per_iter_track0'],4), round(d['ms_per_iter_track1'],4))"
  done
done
