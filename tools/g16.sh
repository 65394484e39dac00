timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "cfg0 or wor_full or wr_full or shards or nodes or full_size_wor" > gpurun_out/g16_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/g16_pytest.log
for a in "2**30 2**20" "2**50 2**24" "2**48 2**32" "2**50 2**10"; do
python tools/debug/one_call.py $a > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -s 0 --csv python tools/debug/one_call.py $a 2>/dev/null | grep -v "^==" > gpurun_out/g16_$(echo $a | tr ' *' '__').csv
done
timeout 300 python tools/sweep.py > gpurun_out/g16_sweep.txt 2>&1; cat gpurun_out/g16_sweep.txt
