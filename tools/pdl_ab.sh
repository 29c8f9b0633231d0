#!/bin/bash
# PDL on/off A/B (1 GPU) + parity suites
o=gpurun_out; tag=${1:-pdl}
b() { timeout 300 python bench.py --config $2 --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$1 $2', round(d['value'],1), round(d['ms_per_step'],4), 'k1', round(d['roofline']['k1_ms'],4), d['clocks']['reasons'])"; }
b pdl cfg2; RK_PDL=0 b nopdl cfg2; b pdl cfg2; RK_PDL=0 b nopdl cfg2
b pdl cfg1; RK_PDL=0 b nopdl cfg1
b pdl cfg3; RK_PDL=0 b nopdl cfg3
timeout 900 python -m pytest tests -m gpu -x -q > $o/${tag}_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $o/${tag}_pytest.log
