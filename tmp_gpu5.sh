B=tools/bin/vb_v1_unroll_sw4_call
$B > gpurun_out/v1_plain.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:MatrixSqrt3x3ELi9EdLi1E -s 0 -c 1 -o gpurun_out/prof_msqrt3_tr $B > gpurun_out/ncu_a.log 2>&1; echo a=$?
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:TrigonometricELi10EdLi0E -s 0 -c 1 -o gpurun_out/prof_trig_nr_v1 $B > gpurun_out/ncu_b.log 2>&1; echo b=$?
