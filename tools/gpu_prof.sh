#!/bin/bash
# ncu --set full captures of chosen jobs: tools/gpu_prof.sh TAG CONFIG BATCH ONLY [more ncu args]
T=$1; CFG=$2; B=$3; ONLY=$4; shift 4
ncu --set full --clock-control none --import-source on -k regex:solve_kernel "$@" -o gpurun_out/${T} \
  python bench.py --config $CFG --batch $B --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline --only "$ONLY" \
  > gpurun_out/${T}_ncu.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/${T}_ncu.log
