WORKLOADS="headline cfg1 wr weak30" bash tools/gpurun_var.sh > gpurun_out/g7_var.txt 2>&1
cat gpurun_out/g7_var.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -k "wor or wr or cta or topup or capacity or cfg or gnm or shards or fullsize or digest or deviates" > gpurun_out/g7_pytest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/g7_pytest.log
