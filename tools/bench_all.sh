#!/bin/bash
# One bench line per BASELINE config on 1 GPU (plus the CPU reference arm for cfg2).
tag=${1:-r01s2}
for c in cfg1 cfg2 cfg3 cfg4 cfg5; do
  timeout 900 python bench.py --config $c > gpurun_out/${tag}_bench_$c.json 2> gpurun_out/${tag}_bench_$c.err
  echo "$c rc=$?"
done
timeout 600 python bench.py --impl reference > gpurun_out/${tag}_bench_reference_cfg2.json 2> gpurun_out/${tag}_bench_reference.err
echo "reference rc=$?"
