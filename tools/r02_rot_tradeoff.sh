#!/bin/bash
# cfg3: accuracy (parity margin) and speed of the Q-rotation period with strip groups.
o=gpurun_out; tag=${1:-r02rt}
timeout 1200 python tools/cfg3_parity_margin.py RK_K1_QROT=2 RK_K1_QROT=3 2>&1 | grep rel
for rep in 1 2; do for v in "RK_K1_GRP=2,RK_K1_QROT=0" "RK_K1_QROT=1" "RK_K1_QROT=2" "RK_K1_QROT=4"; do
  envs=$(echo $v | tr , " ")
  env $envs timeout 600 python bench.py --config cfg3 --steps 30 --warmup 3 --no-cpu --no-e2e --no-secondary > $o/${tag}_${rep}.json 2>/dev/null
  python - $o/${tag}_${rep}.json "$v" <<'PY'
import json,sys
l=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[2], "value %.2f it/s  k1 %.3f ms frac %.3f  clk %s %s"%(l["value"], l["roofline"]["k1_ms"], l["roofline"]["frac"], l["clocks"]["sm_mhz"], l["clocks"]["reasons"]))
PY
done; done
