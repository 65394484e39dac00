./tools/ubench/hgd_lat > gpurun_out/g22_lat.txt 2>&1; cat gpurun_out/g22_lat.txt | grep hgd
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "deviates or cfg0 or wor_full or wr_full or shards" > gpurun_out/g22_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/g22_pytest.log
for a in "2**30 2**20" "2**48 2**32"; do
python tools/debug/one_call.py $a > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -s 0 --csv python tools/debug/one_call.py $a 2>/dev/null | grep -v "^==" > gpurun_out/g22_$(echo $a | tr ' *' '__').csv
done
timeout 300 python tools/sweep.py > gpurun_out/g22_sweep.txt 2>&1; cat gpurun_out/g22_sweep.txt
