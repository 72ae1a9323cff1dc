# Every libpgg kernel under one ncu pass: DRAM bytes + duration per launch
# (the command is run once without ncu first; ncu only if that exited 0)
timeout 600 python tools/all_kernels.py > gpurun_out/all_kernels.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"^k_" --csv --log-file gpurun_out/all_kernels_ncu.csv python tools/all_kernels.py > gpurun_out/all_kernels_ncu.log 2>&1
echo all_kernels=$?
