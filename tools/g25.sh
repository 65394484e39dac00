WORKLOADS="headline cfg1 wr" bash tools/gpurun_var.sh > gpurun_out/g25_var.txt 2>&1
cat gpurun_out/g25_var.txt
