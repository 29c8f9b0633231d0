#!/bin/bash
# Final fresh-box verification (1 GPU): GPU suite, smoke, the default bench line,
# the reference arm, the default command's launch list (first 400 launches), and
# ncu --set full of K1 at cfg3.
tag=${1:-r02f}
o=gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > $o/${tag}_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $o/${tag}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $o/${tag}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python bench.py > $o/${tag}_bench.json 2> $o/${tag}_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > $o/${tag}_bench_ref.json 2> $o/${tag}_bench_ref.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $o/${tag}_launches_default.csv \
    python bench.py --no-cpu --no-e2e --no-secondary > $o/${tag}_ncu_default.log 2>&1; echo "ncu list rc=$?"
timeout 600 python bench.py --config cfg3 --steps 1 --warmup 3 --no-cpu --no-e2e --no-secondary > $o/${tag}_plain3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k1_tc_kernel" -s 2 -c 1 -o $o/${tag}_k1_cfg3 \
    python bench.py --config cfg3 --steps 1 --warmup 3 --no-cpu --no-e2e --no-secondary > $o/${tag}_ncu_f3.log 2>&1; echo "ncu full rc=$?"
