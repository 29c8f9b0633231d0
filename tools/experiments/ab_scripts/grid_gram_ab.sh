#!/bin/bash
# Grid ranks with the tensor-core G/S (sp_gram_tc_k) vs k2a_v4 (RK_GRID_GRAM_TC=0), then the grid checks
N=${1:-2}; tag=${2:-r01s5}; o=gpurun_out
run() { timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $1 "${@:2}"; }
RK_GRID_GRAM_TC=0 run 29580 bench.py --gpus $N --config cfg3 --no-cpu --no-e2e > $o/${tag}_gridoff_bench_cfg3_$N.json 2> $o/${tag}_gridoff_cfg3.err; echo "off cfg3 rc=$?"
RK_GRID_GRAM_TC=0 run 29581 bench.py --gpus $N --config cfg2 --no-cpu --no-e2e > $o/${tag}_gridoff_bench_cfg2_$N.json 2> $o/${tag}_gridoff_cfg2.err; echo "off cfg2 rc=$?"
bash tools/grid_verify.sh $N $tag
for f in $o/${tag}_gridoff_bench_cfg*_$N.json; do python -c "import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);print('$f', round(d['value'],1), d['unit'], d.get('clocks'))" 2>&1 | tail -1; done
