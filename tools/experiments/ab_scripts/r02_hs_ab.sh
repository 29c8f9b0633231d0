#!/bin/bash
# K1 split stages (RK_K1_HS=1) vs whole stages: parity, then interleaved cfg3 / cfg2 timing.
o=gpurun_out
RK_K1_HS=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_north_star.py -x -q -p no:cacheprovider -k "not rescalk" > $o/r02hs_pytest.log 2>&1; echo "pytest hs rc=$?"; tail -2 $o/r02hs_pytest.log
for rep in 1 2; do
  for hs in 0 1; do
    for c in cfg3 cfg2; do
      st=40; [ $c = cfg2 ] && st=300
      RK_K1_HS=$hs timeout 600 python bench.py --config $c --steps $st --warmup 5 --no-cpu --no-e2e --no-secondary > $o/r02hs_${c}_hs${hs}_$rep.json 2>/dev/null
      python - $o/r02hs_${c}_hs${hs}_$rep.json <<'PY'
import json,sys
l=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], "value %.2f k1 %.4f frac %.3f clk %s"%(l["value"], l["roofline"]["k1_ms"], l["roofline"]["frac"], l["clocks"]["sm_mhz"]))
PY
    done
  done
done
