#!/bin/bash
# A/B of a kernel switch: bash tools/env_ab.sh RK_VAR tag — runs tools/k2af_check.py
# with RK_VAR=0 and with the default on several shapes, a cfg2 phase split, then the GPU suite
var=$1; tag=$2; o=gpurun_out/${tag}_ab.log; : > $o
for c in cfg1 k20 cfg2 cfg5 k32m; do
  env $var=0 timeout 300 python tools/k2af_check.py $c >> $o 2>&1
  timeout 300 python tools/k2af_check.py $c >> $o 2>&1
done
timeout 300 python tools/phase_split.py cfg2 >> $o 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest.log 2>&1; echo "pytest rc=$?" >> $o
