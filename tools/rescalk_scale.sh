#!/bin/bash
# RESCALk replicas: 1 vs N GPUs on the same sweep (k_opt and per-k scores must agree)
N=${1:-4}; o=gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -k rescalk -x -q 2>&1 | tail -1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29570 bench.py --gpus $N --config cfg5 --k-min 13 --k-max 16 > $o/rk_cfg5_$N.json 2> $o/rk_cfg5_$N.err; echo "cfg5x$N rc=$?"
timeout 900 python bench.py --config cfg5 --k-min 13 --k-max 16 > $o/rk_cfg5_1.json 2> $o/rk_cfg5_1.err; echo "cfg5x1 rc=$?"
for f in $o/rk_cfg5_1.json $o/rk_cfg5_$N.json; do python -c "import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);print('$f', round(d['value'],1), d['unit'], round(d['seconds'],2), d['k_opt'], json.dumps(d['timing_rank0']))" 2>&1 | tail -1; done
