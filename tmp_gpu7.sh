timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke7.log 2>&1; echo smoke=$?
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu7.log 2>&1; echo pytest=$?
timeout 600 python bench.py --steps 2 --warmup 1 --batch 262144 --e2e-steps 1 --stats gpurun_out/bench7_stats.json > gpurun_out/bench7.log 2>&1; echo bench=$?
