#!/bin/bash
# ncu --set full of chosen jobs, summarised on the box (reports deleted).
#   tools/gpu_prof_list.sh TAG "name config batch only" ...
T=$1; shift
for spec in "$@"; do
  set -- $spec
  name=$1; cfg=$2; b=$3; only=$4
  bash tools/gpu_prof.sh ${T}_$name $cfg $b "$only"
  python tools/ncu_summary.py gpurun_out/${T}_$name.ncu-rep > gpurun_out/${T}_ncu_$name.txt 2>&1
  python tools/ncu_sass_hot.py gpurun_out/${T}_$name.ncu-rep 30 >> gpurun_out/${T}_ncu_$name.txt 2>&1
  ncu -i gpurun_out/${T}_$name.ncu-rep --page source --csv --print-source cuda,sass > /tmp/${T}_${name}_src.csv 2>/dev/null
  python tools/ncu_source_split.py /tmp/${T}_${name}_src.csv 40 >> gpurun_out/${T}_ncu_$name.txt 2>&1
  rm -f gpurun_out/${T}_$name.ncu-rep /tmp/${T}_${name}_src.csv
done
