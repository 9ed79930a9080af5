#!/bin/bash
# ncu --set full + source-line split of chosen C2 jobs:
#   tools/gpu_prof_src.sh TAG name:ONLY [name:ONLY ...]
T=$1; shift
for spec in "$@"; do
  n=${spec%%:*}; only=${spec#*:}
  bash tools/gpu_prof.sh ${T}_$n c2 262144 "$only"
  python tools/ncu_summary.py gpurun_out/${T}_$n.ncu-rep > gpurun_out/${T}_ncu_$n.txt 2>&1
  python tools/ncu_sass_hot.py gpurun_out/${T}_$n.ncu-rep 40 >> gpurun_out/${T}_ncu_$n.txt 2>&1
  ncu -i gpurun_out/${T}_$n.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${T}_${n}_src.csv 2>/dev/null
  python tools/ncu_source_split.py gpurun_out/${T}_${n}_src.csv 60 >> gpurun_out/${T}_ncu_$n.txt 2>&1
  rm -f gpurun_out/${T}_$n.ncu-rep
done
