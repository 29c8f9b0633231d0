#!/bin/bash
# K1 issue-path A/B: warp-uniform elect issue; K=32 merged vs unmerged Q.
o=gpurun_out; tag=${1:-r02k1}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q > $o/${tag}_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $o/${tag}_pytest.log
for mq in 1 0; do
  RK_K1_MERGEQ=$mq timeout 600 python bench.py --config cfg3 --steps 30 --warmup 3 --no-cpu --no-e2e > $o/${tag}_cfg3_mq$mq.json 2>$o/${tag}_cfg3_mq$mq.err
  python - $o/${tag}_cfg3_mq$mq.json <<'PY'
import json,sys
l=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], "value %.2f it/s  k1 %.3f ms frac %.3f  clk %s %s"%(l["value"], l["roofline"]["k1_ms"], l["roofline"]["frac"], l["clocks"]["sm_mhz"], l["clocks"]["reasons"]))
PY
done
timeout 600 python bench.py --config cfg2 --steps 50 --warmup 3 --no-cpu --no-e2e > $o/${tag}_cfg2.json 2>$o/${tag}_cfg2.err
python - $o/${tag}_cfg2.json <<'PY'
import json,sys
l=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], "value %.2f it/s  k1 %.3f ms frac %.3f  clk %s %s"%(l["value"], l["roofline"]["k1_ms"], l["roofline"]["frac"], l["clocks"]["sm_mhz"], l["clocks"]["reasons"]))
PY
