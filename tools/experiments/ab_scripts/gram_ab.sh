#!/bin/bash
# A/B of the dense tensor-core G/S (sp_gram_tc) against k2a_v4, then the GPU suite
o=gpurun_out/gram_ab.log; : > $o
for c in cfg1 k20 cfg2 cfg5; do
  RK_DENSE_GRAM_TC=0 timeout 300 python tools/k2af_check.py $c >> $o 2>&1
  timeout 300 python tools/k2af_check.py $c >> $o 2>&1
done
timeout 300 python tools/phase_split.py cfg2 >> $o 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gram_pytest.log 2>&1; echo "pytest rc=$?" >> $o
