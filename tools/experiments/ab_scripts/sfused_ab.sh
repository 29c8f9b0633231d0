#!/bin/bash
# A/B of the sparse S-fused CSR pass variants (cfg4, 1 GPU)
o=gpurun_out; tag=${1:-ab}
b() { timeout 300 python bench.py --config cfg4 --no-cpu --no-e2e --steps 10 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$1', round(d['value'],1), round(d['ms_per_step'],3), 'k1', round(d['roofline']['k1_ms'],3), d['clocks']['reasons'])"; }
b default
RK_SP_SFUSED=0 b separate
for v in $(ls build/*.so 2>/dev/null); do RK_LIB_PATH=$v b $v; done
