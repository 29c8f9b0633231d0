#!/bin/bash
# sparse grid: parity with either exchange + cfg4 bench / phase split (N GPUs)
N=${1:-2}; tag=${2:-sp}; o=gpurun_out
run() { timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $1 "${@:2}"; }
run 29520 tools/grid_check.py > $o/${tag}_gridcheck_peer_$N.log 2>&1; echo "gridcheck peer rc=$?"; grep -o '"ok": [a-z]*' $o/${tag}_gridcheck_peer_$N.log | head -1
run 29521 bench.py --gpus $N --config cfg4 --no-cpu --no-e2e > $o/${tag}_bench_cfg4_peer_$N.json 2> $o/${tag}_bench_cfg4_peer_$N.err; echo "cfg4 peer rc=$?"
RK_PEER=0 run 29522 bench.py --gpus $N --config cfg4 --no-cpu --no-e2e > $o/${tag}_bench_cfg4_nccl_$N.json 2> $o/${tag}_bench_cfg4_nccl_$N.err; echo "cfg4 nccl rc=$?"
CFG=cfg4 run 29523 tools/grid_overhead.py > $o/${tag}_ovh_peer_$N.log 2>&1; echo "ovh rc=$?"
for f in $o/${tag}_bench_cfg4_*_$N.json; do python -c "import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);print('$f', round(d['value'],1), round(d['ms_per_step'],3), d['config'].get('exchange'))" 2>&1 | tail -1; done
python -c "
import json
d=json.loads([l for l in open('$o/${tag}_ovh_peer_$N.log') if l.startswith('{')][-1])
print([ (round(r['graph_or_direct_ms_per_iter'],3), {k: round(v,3) for k,v in r['phases'].items()}) for r in d['per_rank']])"
