bash tools/gpu_check_stats.sh r02W
bash tools/gpu_sweep.sh r02Wsw dlmin3 | grep -E "trust-region|job"
