#!/bin/bash
# Round evidence on one B200: GPU tests, smoke, the driver's bench commands
# (both arms), every configuration at full size, the ncu launch list of the
# default command and ncu --set full captures of the dominant kernels.
#   tools/gpu_final.sh TAG
T=${1:-final}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/${T}_pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/${T}_smoke.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 --stats gpurun_out/${T}_bench_stats.json > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/${T}_bench_ref.json 2> gpurun_out/${T}_bench_ref.err; echo "ref rc=$?"
python -c "
import json
d=json.load(open('gpurun_out/${T}_bench.json')); r=json.load(open('gpurun_out/${T}_bench_ref.json'))
print('C2', round(d['value']/1e6,2), 'M/s', round(d['ms_per_step'],1), 'ms; e2e', round(d['e2e']['value']/1e6,2), 'M/s; parity', d['parity']['mismatches'], '/', d['parity']['systems'], '; cpu', round(d['cpu_baseline']['value']), '; ref arm', round(r['value']), '; frac', round(d['roofline']['frac'],4), d['clocks'])"
bash tools/gpu_configs.sh ${T} c1 c3 c3f32 c4 c5 n16
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:solve_kernel --csv --log-file gpurun_out/${T}_launches.csv \
  python bench.py --steps 3 --warmup 0 --e2e-steps 0 --no-cpu-baseline > gpurun_out/${T}_ncu_launch.log 2>&1; echo "ncu launches rc=$?"
# ncu --set full captures, summarised on the box (reports are too large to ship back)
prof() {  # name config batch only match bench-kernel-name
  bash tools/gpu_prof.sh ${T}_$1 $2 $3 "$4"
  python tools/ncu_summary.py gpurun_out/${T}_$1.ncu-rep > gpurun_out/${T}_ncu_$1.txt 2>&1
  python tools/ncu_sass_hot.py gpurun_out/${T}_$1.ncu-rep 30 >> gpurun_out/${T}_ncu_$1.txt 2>&1
  ncu -i gpurun_out/${T}_$1.ncu-rep --page source --csv --print-source cuda,sass > /tmp/${T}_$1_src.csv 2>/dev/null
  python tools/ncu_source_split.py /tmp/${T}_$1_src.csv 30 >> gpurun_out/${T}_ncu_$1.txt 2>&1
  NCU_JSON_DIR=gpurun_out python tools/ncu_pipe_json.py gpurun_out/${T}_$1.ncu-rep "$6" $3 "$5"
  rm -f gpurun_out/${T}_$1.ncu-rep /tmp/${T}_$1_src.csv
}
prof c2nr c2 262144 "trigonometric:newton-raphson" "Trigonometric, 10, double, 0" "solve_kernel<test23/trigonometric,n=10,newton-raphson>"
prof c2tr c2 262144 "trigonometric:trust-region" "Trigonometric, 10, double, 1" "solve_kernel<test23/trigonometric,n=10,trust-region>"
prof c2ms c2 262144 "matrix-sqrt-3x3:trust-region" "MatrixSqrt3x3, 9, double, 1" "solve_kernel<test23/matrix-sqrt-3x3,n=9,trust-region>"
prof c1 c1 16777216 "quadratic" "Quadratic<2>, 2, double, 0" "solve_kernel<quadratic,n=2,newton-raphson>"
prof c3 c3 10000000 "klement:n=16" "GeneralizedRosenbrock<16>, 16, double, 3" "solve_kernel<generalized_rosenbrock,n=16,klement>"
prof c4 c4 10000000 "dfsane" "BroydenTridiagonal<16>, 16, double, 4" "solve_kernel<test23/broyden-tridiagonal,n=16,dfsane>"
prof c5 c5 12500000 "dfsane" "Quadratic<4>, 4, double, 4" "solve_kernel<quadratic,n=4,dfsane>"
du -sh gpurun_out
