#!/bin/bash
# Evidence for profiles/: bench lines, launch lists and full ncu captures of the
# dominant kernels (dense cfg2 K1; sparse cfg4 gather pass, numerator, S/G).
tag=${1:-r01}
o=gpurun_out
python bench.py --config cfg2 --steps 3 --warmup 3 --no-cpu --no-e2e > $o/plain2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $o/${tag}_launches_cfg2.csv \
    python bench.py --config cfg2 --steps 3 --warmup 3 --no-cpu --no-e2e > $o/ncu_l2.log 2>&1
python bench.py --config cfg4 --steps 3 --warmup 3 --no-cpu --no-e2e > $o/plain4.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"sp_csr|sp_gram|sp_numer|k2f|emit|wfrag" --csv \
    --log-file $o/${tag}_launches_cfg4.csv python bench.py --config cfg4 --steps 3 --warmup 3 --no-cpu --no-e2e > $o/ncu_l4.log 2>&1
python bench.py --config cfg2 --steps 1 --warmup 3 --no-cpu --no-e2e > $o/plain2b.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k1_tc_kernel" -s 2 -c 1 -o $o/${tag}_k1_cfg2 \
    python bench.py --config cfg2 --steps 1 --warmup 3 --no-cpu --no-e2e > $o/ncu_f2.log 2>&1
python bench.py --config cfg4 --steps 1 --warmup 3 --no-cpu --no-e2e > $o/plain4b.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"sp_csr_pass|sp_numer_tc|sp_gram_tc" -s 6 -c 4 \
    -o $o/${tag}_sparse_cfg4 python bench.py --config cfg4 --steps 1 --warmup 3 --no-cpu --no-e2e > $o/ncu_f4.log 2>&1
echo done
