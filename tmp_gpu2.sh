set -x
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
CMD="python bench.py --steps 1 --warmup 1 --batch 65536 --no-cpu-baseline --e2e-steps 0"
$CMD > gpurun_out/plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo ncu1=$?
$CMD > gpurun_out/plain2.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:TrigonometricELi10EdLi0E -s 1 -c 1 -o gpurun_out/prof_trig_nr $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu2=$?
