#!/bin/bash
# K = 32 merged Q with strip groups: accuracy margin, K1 / k1_reduce (ncu-free bench), power-capped A/B
o=gpurun_out; tag=${1:-r02mq}
timeout 1500 python tools/cfg3_parity_margin.py RK_K1_MERGEQ=1,ITERS=10 RK_K1_MERGEQ=0,ITERS=10 RK_K1_MERGEQ=1,ITERS=30 2>&1 | grep rel
for rep in 1 2 3; do for v in 0 1; do
  RK_K1_MERGEQ=$v timeout 600 python bench.py --config cfg3 --steps 30 --warmup 3 --no-cpu --no-e2e --no-secondary > $o/${tag}_${v}_$rep.json 2>/dev/null
  python - $o/${tag}_${v}_$rep.json $v <<'PY'
import json,sys
l=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print("mergeq", sys.argv[2], "value %.2f it/s  k1 %.3f ms frac %.3f  clk %s %s"%(l["value"], l["roofline"]["k1_ms"], l["roofline"]["frac"], l["clocks"]["sm_mhz"], l["clocks"]["reasons"]))
PY
done; done
