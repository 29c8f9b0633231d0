#!/bin/bash
# Multi-GPU verification (run with gpurun --gpus N): grid parity (small cases and
# the cfg3-size block, both exchanges), the bench line at N (cfg3 strong, self-spawned
# ranks, e2e through solve_on_grid(BlockSource)), cfg2 weak.
o=gpurun_out; tag=${1:-r02m}; N=$(nvidia-smi -L | wc -l)
timeout 2400 python -m pytest tests/test_gpu_grid.py -x -q -p no:cacheprovider > $o/${tag}_grid_pytest_$N.log 2>&1; echo "grid pytest rc=$?"; tail -3 $o/${tag}_grid_pytest_$N.log
for ex in 1 0; do
  RK_PEER=$ex timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29811 tools/grid_check_big.py > $o/${tag}_gridbig_peer${ex}_$N.log 2>&1; echo "gridbig peer=$ex rc=$?"; grep '^{' $o/${tag}_gridbig_peer${ex}_$N.log | cut -c1-400
done
timeout 1800 python bench.py --gpus $N > $o/${tag}_bench_cfg3_$N.json 2> $o/${tag}_bench_cfg3_$N.err; echo "bench cfg3 rc=$?"
timeout 900 python bench.py --gpus $N --config cfg2 --no-e2e > $o/${tag}_bench_cfg2_$N.json 2> $o/${tag}_bench_cfg2_$N.err; echo "bench cfg2 rc=$?"
timeout 900 python bench.py --gpus $N --impl reference --steps 2 --warmup 1 > $o/${tag}_bench_ref_$N.json 2> $o/${tag}_bench_ref_$N.err; echo "ref rc=$?"
for f in $o/${tag}_bench_cfg3_$N.json $o/${tag}_bench_cfg2_$N.json; do python - $f <<'PY'
import json,sys
try:
    l=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[1], "value %.2f it/s e2e %s frac %.3f launches %d clk %s exch %s"%(l["value"], (l.get("e2e") or {}).get("value"), l["roofline"]["frac"], l["gpu_launches"], l["clocks"]["sm_mhz"], l.get("exchange")))
except Exception as e:
    print(sys.argv[1], "parse error", e)
PY
done
