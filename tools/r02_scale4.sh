#!/bin/bash
# 4-GPU verification of the final state: grid parity (4 ranks, both exchanges,
# incl. the cfg3-size block) and the bench at N = 2 and 4 (cfg3 strong, cfg2 weak),
# launched the way the driver does (torchrun) and self-spawned.
o=gpurun_out; tag=${1:-r02s4}
timeout 1800 python -m pytest tests/test_gpu_grid.py -x -q > $o/${tag}_grid_pytest.log 2>&1; echo "grid pytest rc=$?"; tail -2 $o/${tag}_grid_pytest.log
run() { timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $2 "${@:3}"; }
run 4 29581 bench.py --gpus 4 --steps 20 --warmup 3 > $o/${tag}_cfg3_4.json 2> $o/${tag}_cfg3_4.err; echo "cfg3x4 rc=$?"
run 2 29582 bench.py --gpus 2 --steps 20 --warmup 3 > $o/${tag}_cfg3_2.json 2> $o/${tag}_cfg3_2.err; echo "cfg3x2 rc=$?"
run 4 29583 bench.py --gpus 4 --config cfg2 --steps 30 --warmup 3 --no-cpu > $o/${tag}_cfg2_4.json 2> $o/${tag}_cfg2_4.err; echo "cfg2x4 rc=$?"
timeout 900 python bench.py --gpus 4 --config cfg3 --steps 20 --warmup 3 --no-cpu --no-e2e > $o/${tag}_cfg3_4self.json 2> $o/${tag}_cfg3_4self.err; echo "cfg3x4 self-spawn rc=$?"
for f in $o/${tag}_cfg*.json; do python -c "import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);print('$f', round(d['value'],1), d['unit'], d['config']['workload'], 'e2e', (d.get('e2e') or {}).get('value'), 'clk', d['clocks']['sm_mhz'])" 2>&1 | tail -1; done
