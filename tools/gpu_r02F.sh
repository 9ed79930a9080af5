set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02F_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r02F_pytest_gpu.log
bash tools/gpu_configs.sh r02F c3 c1 c5
export NLK_LIB_PATH=paper_2403_16341_b200/libnlk_b200_n2reg.so
bash tools/gpu_configs.sh r02Fn2 c1 c5
timeout 600 python -m pytest tests -m gpu -x -q -k "quadratic or c1 or c5 or boggs or rosenbrock" > gpurun_out/r02Fn2_pytest.log 2>&1; echo "n2 pytest rc=$?"; tail -1 gpurun_out/r02Fn2_pytest.log
