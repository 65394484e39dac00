cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -rf --timeout 300 -x -k "not full_size" > gpurun_out/pytest_a.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_a.log
timeout 900 python -m pytest tests -m gpu -v -rf --timeout 400 --durations=0 -k "full_size" > gpurun_out/pytest_b.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_b.log
timeout 300 python bench.py --steps 10 --warmup 3 --cpu-seconds 5 > gpurun_out/bench3.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench3.log
timeout 300 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/plain3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_leaf|k_split" -c 14 -o gpurun_out/prof3 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu3.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu3.log
