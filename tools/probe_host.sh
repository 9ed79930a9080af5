set -x
lscpu | head -30 > gpurun_out/host_lscpu.txt
nproc >> gpurun_out/host_lscpu.txt
ldd --version | head -1 >> gpurun_out/host_lscpu.txt
python -c "
import numpy as np, json, platform, os
from numpy._core._multiarray_umath import __cpu_features__ as F
print(json.dumps({k:v for k,v in F.items() if v}))
print(platform.libc_ver())
import threadpoolctl
import scipy.linalg
print(json.dumps(threadpoolctl.threadpool_info(), indent=1))
" > gpurun_out/host_np.txt 2>&1
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_start.log 2>&1; echo rc=$?
tail -3 gpurun_out/pytest_gpu_start.log
