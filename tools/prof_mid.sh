export TK_MID_ONLY=1
for k in ${KERNELS:-mid_med_kernel mid_window_kernel mid_scatter_kernel mid_fold_big_kernel}; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -c 1 -f -o gpurun_out/prof_$k python tools/time_mode1.py 400000000 > gpurun_out/prof_$k.log 2>&1
done
ls gpurun_out/
