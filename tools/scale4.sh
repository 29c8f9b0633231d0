#!/bin/bash
# 4-GPU lines not covered elsewhere: sparse cfg4 (2x2 grid) and RESCALk cfg5 replicas (+1-GPU reference point)
o=gpurun_out
run() { timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $1 "${@:2}"; }
run 29560 bench.py --gpus 4 --config cfg4 --no-cpu --no-e2e > $o/s4_cfg4_4.json 2> $o/s4_cfg4_4.err; echo "cfg4x4 rc=$?"
run 29561 bench.py --gpus 4 --config cfg5 --k-min 13 --k-max 16 > $o/s4_cfg5_4.json 2> $o/s4_cfg5_4.err; echo "cfg5x4 rc=$?"
timeout 900 python bench.py --config cfg5 --k-min 13 --k-max 16 > $o/s4_cfg5_1.json 2> $o/s4_cfg5_1.err; echo "cfg5x1 rc=$?"
for f in $o/s4_*.json; do python -c "import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);print('$f', round(d['value'],1), d['unit'], d['config']['workload'], d.get('k_opt'))" 2>&1 | tail -1; done
