N=2; o=gpurun_out; tag=p2
run() { timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $1 "${@:2}"; }
for c in cfg2 cfg3; do
  run 29512 bench.py --gpus $N --config $c --no-cpu --no-e2e > $o/${tag}_bench_${c}_peer_$N.json 2> $o/${tag}_bench_${c}_peer_$N.err; echo "$c peer rc=$?"
done
RK_PROFILE_PHASES=1 run 29514 tools/grid_overhead.py > $o/${tag}_overhead_peer.log 2>&1; echo ovh rc=$?
RK_PEER=0 run 29515 tools/grid_overhead.py > $o/${tag}_overhead_nccl.log 2>&1; echo ovh rc=$?
for f in $o/${tag}_bench_*_$N.json; do echo "== $f"; python -c "import json,sys;d=json.loads(open('$f').read().strip().splitlines()[-1]);print(round(d['value'],1), d['unit'], d['ms_per_step'], d['config'].get('exchange'))" 2>&1 | tail -1; done
tail -5 $o/${tag}_overhead_peer.log $o/${tag}_overhead_nccl.log
