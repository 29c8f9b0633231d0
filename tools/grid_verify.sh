#!/bin/bash
# Multi-GPU check on N GPUs: grid tests, grid parity on both exchanges, bench lines (cfg2 weak, cfg3 strong)
N=${1:-2}; tag=${2:-r01s4}; o=gpurun_out
run() { timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $1 "${@:2}"; }
timeout 900 python -m pytest tests/test_gpu_grid.py -m gpu -q > $o/${tag}_grid_pytest_$N.log 2>&1; echo "grid pytest rc=$?"
run 29570 tools/grid_check.py > $o/${tag}_gridcheck_peer_$N.log 2>&1; echo "gridcheck peer rc=$?"
RK_PEER=0 run 29571 tools/grid_check.py > $o/${tag}_gridcheck_nccl_$N.log 2>&1; echo "gridcheck nccl rc=$?"
run 29572 bench.py --gpus $N --config cfg2 --no-cpu > $o/${tag}_bench_cfg2_$N.json 2> $o/${tag}_bench_cfg2_$N.err; echo "cfg2 rc=$?"
run 29573 bench.py --gpus $N --config cfg3 --no-cpu --no-e2e > $o/${tag}_bench_cfg3_$N.json 2> $o/${tag}_bench_cfg3_$N.err; echo "cfg3 rc=$?"
for f in $o/${tag}_bench_cfg*_$N.json; do python -c "import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);print('$f', round(d['value'],1), d['unit'], d.get('clocks'))" 2>&1 | tail -1; done
