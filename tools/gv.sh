WORKLOADS="headline cfg1 wr" bash tools/gpurun_var.sh > gpurun_out/gv.txt 2>&1; cat gpurun_out/gv.txt
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -k "wor or wr or cta or topup or capacity or cfg or fullsize or full_size or nodes or host or lp" > gpurun_out/gv_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/gv_pytest.log
