#!/bin/bash
# Multi-GPU peer-memory exchange vs NCCL: parity (grid_check) and bench lines.
# usage (on a gpurun --gpus N box): bash tools/peer_check.sh N tag
N=${1:-2}; tag=${2:-peer}; o=gpurun_out
run() { timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $1 "${@:2}"; }
run 29510 tools/grid_check.py > $o/${tag}_gridcheck_peer_$N.log 2>&1; echo "gridcheck peer rc=$?"
RK_PEER=0 run 29511 tools/grid_check.py > $o/${tag}_gridcheck_nccl_$N.log 2>&1; echo "gridcheck nccl rc=$?"
for c in cfg2 cfg3; do
  run 29512 bench.py --gpus $N --config $c --no-cpu --no-e2e > $o/${tag}_bench_${c}_peer_$N.json 2> $o/${tag}_bench_${c}_peer_$N.err; echo "$c peer rc=$?"
  RK_PEER=0 run 29513 bench.py --gpus $N --config $c --no-cpu --no-e2e > $o/${tag}_bench_${c}_nccl_$N.json 2> $o/${tag}_bench_${c}_nccl_$N.err; echo "$c nccl rc=$?"
done
for f in $o/${tag}_gridcheck_*_$N.log; do echo "== $f"; grep -o '"ok": [a-z]*' $f | head -1; grep -o '"exchange": "[a-z]*"' $f | sort | uniq -c; done
for f in $o/${tag}_bench_*_$N.json; do echo "== $f"; python -c "import json,sys;d=json.loads(open('$f').read().strip().splitlines()[-1]);print(round(d['value'],1), d['unit'], d['ms_per_step'], d['config'].get('exchange'))" 2>&1 | tail -1; done
