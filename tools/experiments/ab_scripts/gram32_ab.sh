#!/bin/bash
# A/B of the dense tensor-core G/S at K = 32 (sp_gram_tc_k<32>) against k2a_v4<32>, then the GPU suite
o=gpurun_out/gram32_ab.log; : > $o
for c in k32s k32m cfg3; do
  RK_DENSE_GRAM_TC32=0 timeout 300 python tools/k2af_check.py $c >> $o 2>&1
  timeout 300 python tools/k2af_check.py $c >> $o 2>&1
done
RK_DENSE_GRAM_TC32=0 timeout 300 python tools/phase_split.py cfg3 >> $o 2>&1
timeout 300 python tools/phase_split.py cfg3 >> $o 2>&1
timeout 600 python bench.py --config cfg3 > gpurun_out/gram32_bench_cfg3.json 2>gpurun_out/gram32_bench_cfg3.err
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gram32_pytest.log 2>&1; echo "pytest rc=$?" >> $o
