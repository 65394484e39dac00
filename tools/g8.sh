WORKLOADS="headline cfg1" bash tools/gpurun_var.sh > gpurun_out/g8_var.txt 2>&1
cat gpurun_out/g8_var.txt
