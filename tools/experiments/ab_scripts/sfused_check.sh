#!/bin/bash
# sparse S-fused CSR pass: parity tests + cfg4 bench with / without the fusion
o=gpurun_out; tag=${1:-sf}
timeout 600 python -m pytest tests/test_gpu_sparse.py tests/test_gpu_reference_suite.py -x -q > $o/${tag}_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $o/${tag}_pytest.log
timeout 300 python bench.py --config cfg4 --no-cpu --no-e2e --steps 10 > $o/${tag}_cfg4_fused.json 2> $o/${tag}_cfg4_fused.err; echo "fused rc=$?"
RK_SP_SFUSED=0 timeout 300 python bench.py --config cfg4 --no-cpu --no-e2e --steps 10 > $o/${tag}_cfg4_sep.json 2> $o/${tag}_cfg4_sep.err; echo "sep rc=$?"
for f in $o/${tag}_cfg4_*.json; do python -c "import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);print('$f', round(d['value'],1), round(d['ms_per_step'],3), round(d['roofline']['k1_ms'],3), d['clocks'])"; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"sp_" --csv --log-file $o/${tag}_launches.csv python bench.py --config cfg4 --no-cpu --no-e2e --steps 2 --warmup 3 > /dev/null 2>&1; echo "ncu rc=$?"
python tools/ncu_launches.py $o/${tag}_launches.csv 2>/dev/null | head -12
