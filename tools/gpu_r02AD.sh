bash tools/gpu_check_stats.sh r02AD
timeout 600 python -m pytest tests/test_gpu_defer.py -q > gpurun_out/r02AD_defer.log 2>&1; echo "defer rc=$? $(tail -1 gpurun_out/r02AD_defer.log)"
bash tools/gpu_variants.sh r02ADv "trigonometric:trust" rul5
