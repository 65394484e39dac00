timeout 900 python tools/debug/lp_check.py > gpurun_out/g3_lp.txt 2>&1; echo "lp rc=$?"
cat gpurun_out/g3_lp.txt
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "deviates or wor_full or wr_full or cta_path or capacity or host_stream" > gpurun_out/g3_pytest.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/g3_pytest.log
