#!/bin/bash
# Fused k-wide chain: correctness (bit-identical to the separate kernels, oracle parity) and speed.
o=gpurun_out; tag=${1:-r02c}
timeout 1200 python -m pytest tests/test_gpu_north_star.py tests/test_gpu_parity.py -x -q -p no:cacheprovider > $o/${tag}_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 $o/${tag}_pytest.log
for c in cfg1 cfg2 cfg3; do
  st=30; [ $c = cfg1 ] && st=3000; [ $c = cfg2 ] && st=200
  timeout 600 python bench.py --config $c --steps $st --warmup 5 --no-cpu --no-e2e --no-secondary > $o/${tag}_$c.json 2>$o/${tag}_$c.err
  python - $o/${tag}_$c.json <<'PY'
import json,sys
l=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], "value %.2f it/s  ms/step %.4f k1 %.4f ms frac %.3f launches %d clk %s %s"%(l["value"], l["ms_per_step"], l["roofline"]["k1_ms"], l["roofline"]["frac"], l["gpu_launches"], l["clocks"]["sm_mhz"], l["clocks"]["reasons"]))
PY
done
timeout 300 python bench.py --config cfg2 --steps 3 --warmup 3 --no-cpu --no-e2e --no-secondary > $o/${tag}_plain2.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $o/${tag}_launches_cfg2.csv \
    python bench.py --config cfg2 --steps 3 --warmup 3 --no-cpu --no-e2e --no-secondary > $o/${tag}_ncu_l2.log 2>&1; echo "ncu rc=$?"
