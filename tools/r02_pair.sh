#!/bin/bash
# Paired K1 strips: GPU tests, then cfg3 / cfg2 step and K1 time (HEAD build vs pairs off / on), interleaved.
o=gpurun_out; tag=${1:-r02p}; reps=${2:-2}
timeout 900 python -m pytest tests/test_gpu_north_star.py tests/test_gpu_parity.py tests/test_gpu_guards.py -x -q > $o/${tag}_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $o/${tag}_pytest.log
[ "$(grep -c passed $o/${tag}_pytest.log)" = 0 ] && exit 1
for rep in $(seq $reps); do for cfg in cfg3 cfg2; do for v in head new; do
  case $v in head) envs="RK_LIB_PATH=paper_2202_09512_b200/librescal_b200_head.so";; new) envs="RK_NOTHING=1";; esac
  env $envs timeout 600 python bench.py --config $cfg --steps 30 --warmup 3 --no-cpu --no-e2e --no-secondary > $o/${tag}_${cfg}_${v}_$rep.json 2>$o/${tag}_${cfg}_${v}_$rep.err
  python - $o/${tag}_${cfg}_${v}_$rep.json <<'PY'
import json,sys
l=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], "value %.2f it/s  k1 %.3f ms frac %.3f  clk %s %s"%(l["value"], l["roofline"]["k1_ms"], l["roofline"]["frac"], l["clocks"]["sm_mhz"], l["clocks"]["reasons"]))
PY
done; done; done
