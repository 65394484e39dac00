./tools/ubench/ubench > gpurun_out/g2_ubench.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/g2_pytest.log 2>&1
echo "pytest rc=$?"
tail -25 gpurun_out/g2_pytest.log
python bench.py > gpurun_out/g2_bench.json 2> gpurun_out/g2_bench.err; echo "bench rc=$?"
cat gpurun_out/g2_bench.json
cat gpurun_out/g2_ubench.txt
