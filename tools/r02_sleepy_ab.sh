#!/bin/bash
# K1 epilogue waits: suspend-hint try_wait (default build) vs tight spin (A/B build), cfg3 under the power cap.
o=gpurun_out
for rep in 1 2 3; do
  for v in spin sleepy; do
    if [ $v = spin ]; then lib=$PWD/paper_2202_09512_b200/librescal_b200_spin.so; else lib=$PWD/paper_2202_09512_b200/librescal_b200.so; fi
    RK_LIB_PATH=$lib timeout 600 python bench.py --config cfg3 --steps 60 --warmup 5 --no-cpu --no-e2e --no-secondary > $o/r02sl_${v}_$rep.json 2>/dev/null
    python - $o/r02sl_${v}_$rep.json <<'PY'
import json,sys
l=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], "value %.2f k1 %.3f frac %.3f clk %s"%(l["value"], l["roofline"]["k1_ms"], l["roofline"]["frac"], l["clocks"]["sm_mhz"]))
PY
  done
done
