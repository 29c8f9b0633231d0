#!/bin/bash
# cfg5 as BASELINE names it: the full k = 2..16 sweep, r = 10, on N GPUs and on 1
N=${1:-4}; o=gpurun_out
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29571 bench.py --gpus $N --config cfg5 --k-min 2 --k-max 16 > $o/rkf_cfg5_$N.json 2> $o/rkf_cfg5_$N.err; echo "cfg5x$N rc=$?"
timeout 1200 python bench.py --config cfg5 --k-min 2 --k-max 16 > $o/rkf_cfg5_1.json 2> $o/rkf_cfg5_1.err; echo "cfg5x1 rc=$?"
for f in $o/rkf_cfg5_1.json $o/rkf_cfg5_$N.json; do python -c "import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);t=d['timing_rank0'];print('$f', round(d['value'],1), d['unit'], round(d['seconds'],2), 'k_opt', d['k_opt'], 'upload/members per rank', t.get('upload_members_seconds_per_rank'), 'gather', t.get('gather_seconds'))" 2>&1 | tail -1; done
