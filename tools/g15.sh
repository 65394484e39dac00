./tools/ubench/hgd_lat > gpurun_out/g15_lat.txt 2>&1; cat gpurun_out/g15_lat.txt
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "deviates or cfg0 or wor_full or wr_full or shards" > gpurun_out/g15_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/g15_pytest.log
python tools/debug/one_call.py 2**30 2**20 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -s 0 --csv python tools/debug/one_call.py 2**30 2**20 2>/dev/null | grep -v "^==" > gpurun_out/g15_cfg0.csv
python tools/debug/one_call.py 2**50 2**24 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -s 0 --csv python tools/debug/one_call.py 2**50 2**24 2>/dev/null | grep -v "^==" > gpurun_out/g15_w24.csv
