timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu6.log 2>&1; echo pytest=$?
timeout 600 python bench.py --steps 2 --warmup 1 --batch 262144 --e2e-steps 1 --stats gpurun_out/bench6_stats.json > gpurun_out/bench6.log 2>&1; echo bench=$?
