#!/bin/bash
# Same-input A/B of two library builds: factor hashes after 20 iterations (must match
# bit for bit when a change keeps the arithmetic) and graph-replayed ms/iteration.
for cfg in cfg1 cfg2 k32s cfg3; do
  for lib in old new; do
    if [ $lib = old ]; then L=$PWD/paper_2202_09512_b200/librescal_b200_old.so; else L=$PWD/paper_2202_09512_b200/librescal_b200.so; fi
    RK_LIB_PATH=$L timeout 300 python tools/k2af_check.py $cfg 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$cfg', '$lib', d['hash_track0'], d['hash_track1'], round(d['ms_per_iter_track0'],4))"
  done
done
