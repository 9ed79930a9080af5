timeout 900 python -m pytest tests -m gpu -q -x -k "golden or c1_full or determinism or host_buffer" > gpurun_out/pytest_gpu3.log 2>&1; echo pytest=$?
timeout 600 python bench.py --steps 2 --warmup 1 --batch 262144 --no-cpu-baseline --e2e-steps 1 --stats gpurun_out/bench3_stats.json > gpurun_out/bench3.log 2>&1; echo bench=$?
