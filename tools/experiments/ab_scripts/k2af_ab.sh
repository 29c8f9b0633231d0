#!/bin/bash
# A/B + bit-equality of the fused k2af path (tools/k2af_check.py), then the GPU suite
o=gpurun_out/k2af_ab.log; : > $o
for c in cfg1 k20 k32s cfg2 cfg5 cfg3; do
  RK_K2AF=1 timeout 300 python tools/k2af_check.py $c >> $o 2>  RK_K2AF=0 timeout 300 python tools/k2af_check.py $c >> $o 2>&11
  timeout 300 python tools/k2af_check.py $c >> $o 2>&1
done
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/k2af_pytest.log 2>&1; echo "pytest rc=$?" >> $o
