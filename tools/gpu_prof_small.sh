T=r02w
prof() {
  bash tools/gpu_prof.sh ${T}_$1 $2 $3 "$4"
  python tools/ncu_summary.py gpurun_out/${T}_$1.ncu-rep > gpurun_out/${T}_ncu_$1.txt 2>&1
  python tools/ncu_sass_hot.py gpurun_out/${T}_$1.ncu-rep 30 >> gpurun_out/${T}_ncu_$1.txt 2>&1
  ncu -i gpurun_out/${T}_$1.ncu-rep --page source --csv --print-source cuda,sass > /tmp/${T}_$1_src.csv 2>/dev/null
  python tools/ncu_source_split.py /tmp/${T}_$1_src.csv 30 >> gpurun_out/${T}_ncu_$1.txt 2>&1
  rm -f gpurun_out/${T}_$1.ncu-rep
}
prof ms2 c2 262144 "matrix-sqrt-2x2:trust"
prof brown c2 262144 "brown-almost-linear:newton"
prof boggs c2 262144 "boggs:newton"
