#!/bin/bash
# A/B of the sparse single-GPU K = 32 G/S: tensor-core sp_gram_tc_k<32> against the SIMT sp_gram<32>
o=gpurun_out/sp_gram32_ab.log; : > $o
RK_SP_GRAM_SIMT=1 timeout 600 python tools/phase_split.py cfg4k32 >> $o 2>&1
timeout 600 python tools/phase_split.py cfg4k32 >> $o 2>&1
timeout 900 python -m pytest tests/test_gpu_sparse.py tests/test_gpu_parity.py -x -q > gpurun_out/sp_gram32_pytest.log 2>&1; echo "pytest rc=$?" >> $o
