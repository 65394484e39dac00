set -x
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 500 > gpurun_out/g1_clocks.csv &
CK=$!
./tools/ubench/ubench > gpurun_out/g1_ubench.txt 2>&1
kill $CK
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -x -q -rA --durations=0 > gpurun_out/g1_fullsize.log 2>&1
echo "pytest rc=$?"
tail -30 gpurun_out/g1_fullsize.log
cat gpurun_out/g1_ubench.txt
nproc
