timeout 600 python -m pytest tests/test_gpu_sparse.py -x -q 2>&1 | tail -2
python bench.py --config cfg4 --no-cpu --no-e2e --steps 3 --warmup 3 > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"sp_csr|sp_gram|sp_numer|k2f|emit|set_tail" --csv --log-file gpurun_out/launches_cfg4.csv python bench.py --config cfg4 --no-cpu --no-e2e --steps 3 --warmup 3 > gpurun_out/ncu.log 2>&1
python bench.py --config cfg4 --no-cpu --no-e2e --steps 10 | cut -c1-400
