#!/bin/bash
# One GPU round trip: GPU tests, smoke, a short bench with the parity leg.
#   tools/gpu_check.sh TAG [bench args...]
TAG=${1:-x}; shift
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/${TAG}_pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"
tail -2 gpurun_out/${TAG}_smoke.log
timeout 900 python bench.py --stats gpurun_out/${TAG}_bench_stats.json "$@" > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
tail -c 600 gpurun_out/${TAG}_bench.json
